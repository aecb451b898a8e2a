"""One exact K-Means C3 region launch (16M x 32 x 64) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n = int(os.environ.get("N", 1 << 24)); d, k = 32, 64
pts = E.make_blobs(n, d, k, 42, 30.0)
grid, mp = E.resolve_grid("kmeans", n, items_per_thread=4)
dp = torch.from_numpy(pts).cuda(); dc = torch.from_numpy(pts[:k].copy()).cuda()
lab = torch.zeros(n, dtype=torch.int32, device="cuda")
print(E.run_region(grid, n, mp, E.kmeans_region(dp, dc, lab), None).kernel_ms)
