"""Probe: K-Means Lloyd loop, random perforation at thread / warp / team level."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n, d, k = 1 << 24, 32, 64
pts = E.make_blobs(n, d, k, 42, 30.0)
grid, _ = E.resolve_grid("kmeans", n, items_per_thread=4)
dp = torch.from_numpy(pts).cuda(); c0 = torch.from_numpy(pts[:k].copy()).cuda()
ex = E.kmeans_run(grid, dp, k, None, max_iters=40, centroids=c0.clone())
ex = E.kmeans_run(grid, dp, k, None, max_iters=40, centroids=c0.clone())
te = ex.region_ms + ex.update_ms
print(f"exact: {te:.1f} ms  region {ex.region_ms:.1f} update {ex.update_ms:.1f} iters {ex.iterations}")
for lv in os.environ.get("LEVELS", "thread,warp,team").split(","):
    for p in ((50, 75) if lv != "team" else (52, 54, 56, 58)):
        sp = E.perfo("random", p, level=lv)
        r = E.kmeans_run(grid, dp, k, sp, max_iters=40, centroids=c0.clone(), perfo_seed_base=7)
        r = E.kmeans_run(grid, dp, k, sp, max_iters=40, centroids=c0.clone(), perfo_seed_base=7)
        t = r.region_ms + r.update_ms
        print(f"{lv:6s} p={p}: {t:.1f} ms (x{te / t:.3f}) region {r.region_ms:.1f} rate {r.stats['approx_invocations'] / r.stats['total_invocations']:.3f} "
              f"mcr {E.mcr(ex.assignments, r.assignments):.4f} iters {r.iterations}")
