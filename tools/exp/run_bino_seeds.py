"""Probe: headline binomial config's MAPE across the per-rank seeds (42 + rank)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n = 1 << 20
grid, mp = E.resolve_grid("binomial", n, items_per_thread=384)
for seed in range(42, 50):
    d = torch.from_numpy(E.make_binomial_portfolio(n, seed)).cuda()
    ex = torch.zeros(n, dtype=torch.float64, device="cuda"); out = torch.zeros_like(ex)
    E.run_region(grid, n, mp, E.binomial_region(d, 1024, ex), None)
    b = E.run_region(grid, n, mp, E.binomial_region(d, 1024, out), E.iact(4, 0.4, level="team"))
    print(seed, f"rate {b.approx_rate():.3f} mape {E.mape(ex, out):.5f}", flush=True)
