"""C3 Lloyd loop (16 M x 32 x 64, separation 30, perfo(random:52) level(team), 40 iterations):
region / update time split as the library reports it."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n = int(os.environ.get("N", 1 << 24)); d, k = 32, 64
pts = E.make_blobs(n, d, k, 42, 30.0)
grid, _ = E.resolve_grid("kmeans", n, items_per_thread=4)
dp = torch.from_numpy(pts).cuda(); c0 = torch.from_numpy(pts[:k].copy()).cuda()
spec = E.perfo("random", 52, level="team", seed=7)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = E.kmeans_run(grid, dp, k, spec, max_iters=40, centroids=c0.clone())
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"iters {r.iterations} wall {t*1e3:.1f} ms region {r.region_ms:.2f} ms update {r.update_ms:.2f} ms", flush=True)
