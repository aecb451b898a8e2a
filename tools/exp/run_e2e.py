"""Probe: where does the host-buffer (end-to-end) Blackscholes call spend time?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
h_in = torch.from_numpy(opts).pin_memory(); h_out = torch.zeros(n, dtype=torch.float64).pin_memory()
reg = E.blackscholes_region(h_in.numpy(), h_out.numpy())
spec = E.taf(5, 1, 0.5)
for i in range(4):
    t0 = time.perf_counter(); E.run_region_host(grid, n, mp, reg, spec); t = time.perf_counter() - t0
    print(f"run_region_host pinned: {t*1e3:.2f} ms")
p_in = opts.copy(); p_out = np.zeros(n)
reg2 = E.blackscholes_region(p_in, p_out)
for i in range(2):
    t0 = time.perf_counter(); E.run_region_host(grid, n, mp, reg2, spec); t = time.perf_counter() - t0
    print(f"run_region_host pageable: {t*1e3:.2f} ms")
d = torch.empty(n * 5, dtype=torch.float64, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h_in.view(-1), non_blocking=True); torch.cuda.synchronize()
    print(f"torch H2D 168MB pinned: {(time.perf_counter()-t0)*1e3:.2f} ms")
