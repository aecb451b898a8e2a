"""Profiling driver: LavaMD region, exact then TAF warp (one launch each)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
b1 = int(os.environ.get("B1", 32)); P = 128
n = b1 ** 3
rv, qv = E.make_lavamd(b1, P, 42)
grid, mp = E.resolve_grid("lavamd", n)
d_rv = torch.from_numpy(rv).cuda(); d_qv = torch.from_numpy(qv).cuda()
fv = torch.zeros((n * P, 4), dtype=torch.float64, device="cuda")
spec = E.taf(3, 8, 0.1, os.environ.get("LEVEL", "warp"))
for _ in range(int(os.environ.get("REPS", "1"))):
    fv.zero_(); a = E.run_region(grid, n, mp, E.lavamd_region(d_rv, d_qv, fv, b1, P), None)
    fv.zero_(); b = E.run_region(grid, n, mp, E.lavamd_region(d_rv, d_qv, fv, b1, P), spec)
    print(f"exact {a.kernel_ms:.2f} ms  taf {b.kernel_ms:.2f} ms rate {b.approx_rate():.3f}")
