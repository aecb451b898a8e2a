"""Probe: Binomial 1M x 1024 team iACT at several items-per-thread / thresholds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n = 1 << 20
opts = E.make_binomial_portfolio(n, 42)
d = torch.from_numpy(opts).cuda()
ex = torch.zeros(n, dtype=torch.float64, device="cuda")
for ipt in [int(v) for v in os.environ.get('IPTS', '128,192,256,384').split(',')]:
    grid, mp = E.resolve_grid("binomial", n, items_per_thread=ipt)
    E.run_region(grid, n, mp, E.binomial_region(d, 1024, ex), None)
    a = E.run_region(grid, n, mp, E.binomial_region(d, 1024, ex), None)
    for ts, thr in [(4, float(t)) for t in os.environ.get('THRS', '0.5,0.4').split(',')]:
        out = torch.zeros(n, dtype=torch.float64, device="cuda")
        b = E.run_region(grid, n, mp, E.binomial_region(d, 1024, out), E.iact(ts, thr, level="team"))
        print(f"ipt {ipt} tsize {ts} thr {thr}: exact {a.kernel_ms:.1f} ms approx {b.kernel_ms:.1f} ms "
              f"x{a.kernel_ms / b.kernel_ms:.3f} rate {b.approx_rate():.3f} mape {E.mape(ex, out):.5f}", flush=True)
