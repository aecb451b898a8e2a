"""K-Means C3 region (16M x 32 x 64): DMMA warp filter vs per-lane CUDA-core
filter, exact and team-perforated; labels must agree."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n = int(os.environ.get("N", 1 << 24)); d, k = 32, 64
pts = E.make_blobs(n, d, k, 42, 30.0)
grid, mp = E.resolve_grid("kmeans", n, items_per_thread=4)
dp = torch.from_numpy(pts).cuda(); dc = torch.from_numpy(pts[:k].copy()).cuda()
res = {}
for mode in ("0", "1"):
    os.environ["HPAC_KM_DMMA"] = mode
    lab = torch.zeros(n, dtype=torch.int32, device="cuda")
    ts, tp = [], []
    for _ in range(4):
        ts.append(E.run_region(grid, n, mp, E.kmeans_region(dp, dc, lab), None).kernel_ms)
    l0 = lab.clone()
    for _ in range(4):
        tp.append(E.run_region(grid, n, mp, E.kmeans_region(dp, dc, lab), E.perfo("random", 52, level="team", seed=3)).kernel_ms)
    res[mode] = l0
    print(f"dmma={mode} exact {min(ts[1:]):.3f} ms  random52-team {min(tp[1:]):.3f} ms", flush=True)
print("labels equal:", bool(torch.equal(res["0"], res["1"])))
