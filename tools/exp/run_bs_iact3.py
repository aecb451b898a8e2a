"""Blackscholes C1 shape (4M, 4096x64, ipt 16): exact, TAF, and iACT on the
decide-then-price engine vs the lockstep engine (HPAC_ENGINE=thread)."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if len(sys.argv) == 1:
    for eng in ["auto", "thread"]:
        subprocess.run([sys.executable, __file__, eng], env=dict(os.environ, HPAC_ENGINE=eng))
    sys.exit(0)
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
d = torch.from_numpy(opts).cuda()
ex = torch.zeros(n, dtype=torch.float64, device="cuda"); out = torch.zeros_like(ex)
def t(spec, o, reps=20):
    ms = [E.run_region(grid, n, mp, E.blackscholes_region(d, o), spec).kernel_ms for _ in range(reps)]
    lr = E.run_region(grid, n, mp, E.blackscholes_region(d, o), spec)
    return float(np.median(ms)) * 1e3, lr
te, _ = t(None, ex)
print(f"[{sys.argv[1]}] exact {te:.1f} us")
a = ex.cpu().numpy()
for lvl in ["thread", "warp", "team"]:
    for ts, th in [(2, 0.5), (4, 0.3), (8, 0.3)]:
        ta, lr = t(E.iact(ts, th, level=lvl), out)
        b = out.cpu().numpy(); mape = float(np.mean(np.abs(a - b) / np.abs(a)))
        print(f"[{sys.argv[1]}] iact({ts},{th},{lvl:6s}) {ta:7.1f} us  speedup {te/ta:5.2f}  rate {lr.approx_rate():.3f}  mape {mape*100:.2f}%", flush=True)
