"""Time the exact binomial region (1M options x 1024 steps) for the library
at $HPAC_LIB (tuning helper; prints one JSON line)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_16877_b200 import engine as E
n = int(os.environ.get("N", 1 << 20)); steps = int(os.environ.get("LAT", 1024))
opts = E.make_binomial_portfolio(n, 42)
grid, mp = E.resolve_grid("binomial", n, items_per_thread=128)
d = torch.from_numpy(opts).cuda(); out = torch.zeros(n, dtype=torch.float64, device="cuda")
spec = E.iact(4, 0.5, level="team") if os.environ.get("IACT") else None
E.run_region(grid, n, mp, E.binomial_region(d, steps, out), spec)
lrs = [E.run_region(grid, n, mp, E.binomial_region(d, steps, out), spec) for _ in range(3)]
ts = [lr.kernel_ms for lr in lrs]
print(json.dumps({"lib": os.environ.get("HPAC_LIB"), "ms": min(ts), "Mopt_s": n / min(ts) / 1e3, "iact": bool(spec),
                  "fallbacks": lrs[0].stats["lattice_fallbacks"]}))
