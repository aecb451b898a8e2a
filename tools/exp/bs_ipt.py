"""Blackscholes exact / TAF kernel time vs items per thread (grid shape)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
d = torch.from_numpy(opts).cuda(); o = torch.zeros(n, dtype=torch.float64, device="cuda")
for ipt in [1, 2, 4, 8, 16, 32]:
    grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=ipt)
    for name, spec in [("exact", None), ("taf", E.taf(5, 1, 0.5))]:
        ms = [E.run_region(grid, n, mp, E.blackscholes_region(d, o), spec).kernel_ms for _ in range(20)]
        print(f"ipt {ipt:3d} teams {grid.num_teams:6d} {name:5s} {np.median(ms)*1e3:7.1f} us", flush=True)
