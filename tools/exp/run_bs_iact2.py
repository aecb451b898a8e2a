"""Blackscholes C1 shape: exact / TAF / iACT kernel times (deferred and
lockstep iACT), MAPE vs exact."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
d = torch.from_numpy(opts).cuda()
ex = torch.zeros(n, dtype=torch.float64, device="cuda"); out = torch.zeros_like(ex)
def t(spec, o, reps=20):
    ms = []
    for _ in range(reps):
        lr = E.run_region(grid, n, mp, E.blackscholes_region(d, o), spec); ms.append(lr.kernel_ms)
    return float(np.median(ms)) * 1e3, lr
te, _ = t(None, ex)
print(f"exact {te:.1f} us")
specs = [("taf(5,1,0.5)", lambda: E.taf(5, 1, 0.5))]
for lvl in ["thread", "warp", "team"]:
    specs += [(f"iact(2,0.5,{lvl})", lambda lvl=lvl: E.iact(2, 0.5, level=lvl)),
              (f"iact(4,0.3,{lvl})", lambda lvl=lvl: E.iact(4, 0.3, level=lvl))]
for name, f in specs:
    for dv in (["1", "0"] if "iact" in name else ["1"]):
        os.environ["HPAC_IACT_DEFER"] = dv
        ta, lr = t(f(), out)
        a = ex.cpu().numpy(); b = out.cpu().numpy()
        mape = float(np.mean(np.abs(a - b) / np.abs(a)))
        print(f"{name:18s} defer={dv} {ta:7.1f} us  speedup {te/ta:5.2f}  rate {lr.approx_rate():.3f}  mape {mape*100:.2f}%", flush=True)
