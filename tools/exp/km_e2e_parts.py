"""Where the K-Means e2e time goes: pinned H2D of the points, the Lloyd loop
(wall vs kernel time), the label D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n, d, k = 1 << 24, 32, 64
pts = E.make_blobs(n, d, k, 42, 30.0)
grid, _ = E.resolve_grid("kmeans", n, items_per_thread=4)
h = torch.from_numpy(pts).pin_memory()
buf = torch.empty((n, d), dtype=torch.float64, device="cuda")
c0 = buf[:k].clone()
spec = E.perfo("random", 52, level="team")
def wall(f):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize(); return (time.perf_counter() - t) * 1e3, r
for _ in range(2):
    t_h2d, _ = wall(lambda: buf.copy_(h, non_blocking=True))
    c0 = buf[:k].clone()
    t_run, r = wall(lambda: E.kmeans_run(grid, buf, k, spec, max_iters=40, centroids=c0.clone(), perfo_seed_base=7))
    print(f"h2d {t_h2d:.1f} ms ({n*d*8/t_h2d/1e6:.1f} GB/s)  lloyd wall {t_run:.1f} ms  kernels {r.region_ms + r.update_ms:.1f} ms  iters {r.iterations}", flush=True)
# the bench's e2e loop verbatim (events on the current stream)
stream = torch.cuda.current_stream()
h_lab = torch.empty(n, dtype=torch.int32).pin_memory()
buf2 = torch.empty_like(buf)
for rep in range(2):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ev0.record(stream)
    its = 0
    for _ in range(2):
        buf2.copy_(h, non_blocking=True)
        r = E.kmeans_run(grid, buf2, k, spec, max_iters=40, centroids=c0.clone(), perfo_seed_base=7, stream=stream)
        h_lab.copy_(r.assignments, non_blocking=True)
        its += r.iterations
    ev1.record(stream)
    torch.cuda.synchronize()
    print(f"bench-style e2e: events {ev0.elapsed_time(ev1):.1f} ms wall {(time.perf_counter()-t0)*1e3:.1f} ms its {its}", flush=True)
