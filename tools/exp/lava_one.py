"""One LavaMD 64^3 x 128 exact launch (HPAC_LAVA_TILE selects the box order)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
b1, P = 64, 128
nb = b1 ** 3
rv, qv = E.make_lavamd(b1, P, 42)
fv = torch.zeros((nb * P, 4), dtype=torch.float64, device="cuda")
E.run_region(E.GridConfig(nb, P, 32, 1), nb, 1,
             E.lavamd_region(torch.from_numpy(rv).cuda(), torch.from_numpy(qv).cuda(), fv, b1, P), None)
