"""Profiling driver: Blackscholes 4M exact vs iACT (warp level)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
d = torch.from_numpy(opts).cuda(); out = torch.zeros(n, dtype=torch.float64, device="cuda")
sp = E.iact(4, 0.3, level=os.environ.get("LEVEL", "warp"))
for _ in range(int(os.environ.get("REPS", "1"))):
    a = E.run_region(grid, n, mp, E.blackscholes_region(d, out), None)
    b = E.run_region(grid, n, mp, E.blackscholes_region(d, out), sp)
    print(f"exact {a.kernel_ms*1e3:.1f} us  iact {b.kernel_ms*1e3:.1f} us rate {b.approx_rate():.3f}")
