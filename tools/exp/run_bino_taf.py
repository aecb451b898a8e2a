"""Binomial TAF (American puts, per-team, 8 teams per CTA): kernel medians at 256 K options x 1024 steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
n = 1 << 18
opts = E.make_binomial_portfolio(n, 42)
grid, mp = E.resolve_grid("binomial", n, items_per_thread=64)
d = torch.from_numpy(opts).cuda(); o = torch.zeros(n, dtype=torch.float64, device="cuda")
for name, spec in [("taf(5,1,0.5) team", E.taf(5, 1, 0.5, "team")), ("taf(2,4,0.5) team", E.taf(2, 4, 0.5, "team"))]:
    ms = [E.run_region(grid, n, mp, E.binomial_region(d, 1024, o), spec).kernel_ms for _ in range(5)]
    print(f"{name:20s} {np.median(ms):8.2f} ms", flush=True)
