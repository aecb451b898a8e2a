"""Probe: K-Means e2e step (H2D points + Lloyd run + D2H labels) timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n, d, k = 1 << 24, 32, 64
pts = E.make_blobs(n, d, k, 42, 30.0)
grid, _ = E.resolve_grid("kmeans", n, items_per_thread=4)
c0 = torch.from_numpy(pts[:k].copy()).cuda()
h = torch.from_numpy(pts).pin_memory(); buf = torch.empty((n, d), dtype=torch.float64, device="cuda")
lab = torch.empty(n, dtype=torch.int32).pin_memory()
sp = E.perfo("random", 52, level="team")
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    buf.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    r = E.kmeans_run(grid, buf, k, sp, max_iters=40, centroids=c0.clone(), perfo_seed_base=7)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    lab.copy_(r.assignments, non_blocking=True); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"h2d {1e3*(t1-t0):.1f} ms run {1e3*(t2-t1):.1f} ms (device {r.region_ms + r.update_ms:.1f}) d2h {1e3*(t3-t2):.1f} ms")
