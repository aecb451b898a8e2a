"""One Blackscholes C1 launch (warm-up launch first): SPEC=exact|taf|perfo."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=int(os.environ.get("IPT", "16")))
d = torch.from_numpy(opts).cuda(); o = torch.zeros(n, dtype=torch.float64, device="cuda")
spec = {"exact": None, "taf": E.taf(5, 1, 0.5), "perfo": E.perfo("small", 4),
        "iact": E.iact(int(os.environ.get("TSIZE", "2")), 0.5)}[os.environ.get("SPEC", "exact")]
for _ in range(2):
    lr = E.run_region(grid, n, mp, E.blackscholes_region(d, o), spec)
print(lr.kernel_ms)
