"""Binomial C2 grid (1M x 1024, ipt 384) under TAF: 8-teams-per-CTA kernel vs
the one-team-per-CTA path (HPAC_BINO_PIPELINE=0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
n, N = 1 << 20, 1024
opts = E.make_binomial_portfolio(n, 42)
grid, mp = E.resolve_grid("binomial", n, items_per_thread=384)
d = torch.from_numpy(opts).cuda(); o = torch.zeros(n, dtype=torch.float64, device="cuda")
for pipe in ["1", "0"]:
    os.environ["HPAC_BINO_PIPELINE"] = pipe
    for name, spec in [("exact", None), ("taf(5,1,0.5)", E.taf(5, 1, 0.5, "team"))]:
        lr = E.run_region(grid, n, mp, E.binomial_region(d, N, o), spec)
        print(f"pipeline={pipe} {name:14s} {lr.kernel_ms:8.2f} ms  {n / lr.kernel_ms / 1e3:7.2f} M options/s  rate {lr.approx_rate():.3f}", flush=True)
