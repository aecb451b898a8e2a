"""Blackscholes region reading its options from / writing its prices to
pinned host memory directly (UVA zero-copy) vs H2D + kernel + D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
h_in = torch.from_numpy(opts).pin_memory()
h_out = torch.zeros(n, dtype=torch.float64).pin_memory()
d_in = h_in.cuda(); d_out = torch.zeros(n, dtype=torch.float64, device="cuda")
spec = E.taf(5, 1, 0.5)
ref = E.run_region(grid, n, mp, E.blackscholes_region(d_in, d_out), spec)
want = d_out.cpu()
def timeit(f, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    return min(ts) * 1e3
def copy_path():
    d_in.copy_(h_in, non_blocking=True)
    E.run_region(grid, n, mp, E.blackscholes_region(d_in, d_out), spec)
    h_out.copy_(d_out, non_blocking=True)
def zero_copy():
    return E.run_region(grid, n, mp, E.blackscholes_region(h_in, h_out), spec)
print(f"copy path {timeit(copy_path):.3f} ms")
for eng in ("", "thread"):
    os.environ["HPAC_ENGINE"] = eng
    h_out.zero_()
    r = zero_copy()
    ok = torch.equal(h_out, want)
    print(f"zero-copy engine={eng or 'stream'}: {timeit(zero_copy):.3f} ms kernel {r.kernel_ms:.3f} ms equal={ok}")
