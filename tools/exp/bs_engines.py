"""Blackscholes 4M region: stream engine (bulk-TMA tiles) vs generic per-thread
engine, exact and TAF."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = torch.from_numpy(E.make_bs_portfolio(n, 42)).cuda()
out = torch.zeros(n, dtype=torch.float64, device="cuda")
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
for eng in ("", "thread"):
    os.environ["HPAC_ENGINE"] = eng
    for name, spec in (("exact", None), ("taf", E.taf(5, 1, 0.5))):
        ts = [E.run_region(grid, n, mp, E.blackscholes_region(opts, out), spec).kernel_ms for _ in range(8)]
        print(f"{eng or 'stream':6s} {name:5s} {min(ts[2:]) * 1e3:.1f} us", flush=True)
