import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
n = 48
opts = E.make_binomial_portfolio(n, 7)
d = torch.from_numpy(opts).cuda()
for N in [1055, 1056, 1500]:
    for pipe in ["1", "0"]:
        os.environ["HPAC_BINO_PIPELINE"] = pipe
        o = torch.zeros(n, dtype=torch.float64, device="cuda")
        lr = E.run_region(E.GridConfig(n, 64, 32, 1), n, 1, E.binomial_region(d, N, o), None)
        print(N, pipe, o.cpu().numpy()[:4], lr.stats["total_invocations"])
