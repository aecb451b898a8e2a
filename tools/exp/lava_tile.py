"""LavaMD 64^3 x 128 exact: tiled vs natural box order (kernel time)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
b1, P = 64, 128
nb = b1 ** 3
rv, qv = E.make_lavamd(b1, P, 42)
d_rv, d_qv = torch.from_numpy(rv).cuda(), torch.from_numpy(qv).cuda()
fv = torch.zeros((nb * P, 4), dtype=torch.float64, device="cuda")
grid = E.GridConfig(nb, P, 32, 1)
for tile in ["1", "0", "1", "0"]:
    os.environ["HPAC_LAVA_TILE"] = tile
    ms = []
    for _ in range(3):
        fv.zero_()
        ms.append(E.run_region(grid, nb, 1, E.lavamd_region(d_rv, d_qv, fv, b1, P), None).kernel_ms)
    print(f"tile={tile} {np.median(ms):.2f} ms", flush=True)
