"""Lloyd loop wall / event time: CUDA-graph loop vs host-driven loop."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n, d, k = 1 << 24, 32, 64
pts = torch.from_numpy(E.make_blobs(n, d, k, 42, 30.0)).cuda()
grid, _ = E.resolve_grid("kmeans", n, items_per_thread=4)
for name, spec in (("exact", None), ("random52-team", E.perfo("random", 52, level="team"))):
    for host in (False, True, False, True):
        c0 = pts[:k].clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter(); e0.record()
        r = E.kmeans_run(grid, pts, k, spec, max_iters=40, centroids=c0, perfo_seed_base=7, host_loop=host)
        e1.record(); torch.cuda.synchronize(); w = (time.perf_counter() - t) * 1e3
        print(f"{name:14s} host_loop={host!s:5s} graph={r.graph!s:5s} iters {r.iterations} wall {w:7.1f} ms "
              f"events {e0.elapsed_time(e1):7.1f} ms kernels {r.region_ms + r.update_ms:7.1f} ms", flush=True)
