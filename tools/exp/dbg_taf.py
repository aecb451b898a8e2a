import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
from gpu_util import dev
steps, ipt = 32, 24
n = 20 * ipt
opts = E.make_binomial_portfolio(n, 42)
d = dev(opts)
grid, mapping = E.resolve_grid("binomial", n, items_per_thread=ipt)
def run(spec):
    o = torch.zeros(n, dtype=torch.float64, device="cuda"); pa = torch.zeros(n, dtype=torch.uint8, device="cuda")
    lr = E.run_region(grid, n, mapping, E.binomial_region(d, steps, o), spec, paths=pa)
    return o.cpu().numpy(), pa.cpu().numpy()
ex, _ = run(None)
ex2, _ = run(None)
print("exact deterministic:", np.array_equal(ex, ex2))
t, tp = run(E.taf(2, 4, 0.01, "team"))
acc = tp == 0
bad = np.nonzero(acc & (t != ex))[0]
print("accurate steps differing:", len(bad), bad[:10], (t[bad] - ex[bad])[:5])
