"""Points that change label per Lloyd iteration at the C3 shape (what the
incremental centroid update has to move)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n, d, k = 1 << 24, 32, 64
pts = torch.from_numpy(E.make_blobs(n, d, k, 42, float(os.environ.get("SEP", 30.0)))).cuda()
grid, _ = E.resolve_grid("kmeans", n, items_per_thread=4)
spec = E.perfo("random", 52, level="team") if os.environ.get("PERFO") else None
prev = None
for it in range(1, 13):
    r = E.kmeans_run(grid, pts, k, spec, max_iters=it, centroids=pts[:k].clone(), perfo_seed_base=7)
    a = r.assignments.clone()
    ch = n if prev is None else int((a != prev).sum())
    print(f"iter {it:2d}: changed {ch:9d} ({ch / n * 100:.3f} %)  update total {r.update_ms:.2f} ms", flush=True)
    prev = a
