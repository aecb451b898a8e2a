import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
d = np.load("tests/golden/apps.npz"); b = d["bino"]
for steps in (16, 128, 1024):
    o = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    lr = E.run_region(E.GridConfig(len(b), 64, 32, 1), len(b), 1, E.binomial_region(torch.from_numpy(b).cuda(), steps, o), None)
    w = d[f"bino_price_{steps}"]; g = o.cpu().numpy()
    bad = np.where(~(np.abs(g - w) <= 1e-6 * np.abs(w)))[0]
    print(steps, "bad", bad.tolist(), "fallbacks", lr.stats["lattice_fallbacks"])
    for i in bad[:5]:
        S, K, r, v, T = b[i]
        print("  ", i, b[i].tolist(), "gpu", g[i], "want", w[i])
