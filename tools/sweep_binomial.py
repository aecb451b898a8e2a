"""Approximation-parameter sweep for the headline region (Binomial 1M x 1024,
team-shared iACT): items/s, speedup over the exact kernel, MAPE, approx rate.
One JSON line per point; used to pick bench.py's default directive."""
import itertools, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_16877_b200 import engine as E
n = int(os.environ.get("N", 1 << 20)); lat = int(os.environ.get("LAT", 1024))
opts = E.make_binomial_portfolio(n, 42)
d = torch.from_numpy(opts).cuda()
exact = torch.zeros(n, dtype=torch.float64, device="cuda")
g0, mp = E.resolve_grid("binomial", n)
E.run_region(g0, n, mp, E.binomial_region(d, lat, exact), None)
t_exact = min(E.run_region(g0, n, mp, E.binomial_region(d, lat, exact), None).kernel_ms for _ in range(2))
print(json.dumps({"exact_ms": t_exact, "n": n, "lattice": lat}), flush=True)
out = torch.zeros_like(exact)
ipts = [int(x) for x in os.environ.get("IPTS", "32,64,96,128,192,256").split(",")]
thrs = [float(x) for x in os.environ.get("THRS", "0.25,0.5,0.75,1.0").split(",")]
sizes = [int(x) for x in os.environ.get("SIZES", "2,4,8").split(",")]
for ipt, thr, ts in itertools.product(ipts, thrs, sizes):
    g, mp = E.resolve_grid("binomial", n, items_per_thread=ipt)
    spec = E.iact(ts, thr, level="team")
    lr = E.run_region(g, n, mp, E.binomial_region(d, lat, out), spec)
    ms = min(lr.kernel_ms, E.run_region(g, n, mp, E.binomial_region(d, lat, out), spec).kernel_ms)
    print(json.dumps({"ipt": ipt, "thr": thr, "tsize": ts, "ms": ms, "speedup": t_exact / ms,
                      "mape": E.mape(exact, out), "rate": lr.approx_rate(),
                      "Mopt_s": n / ms / 1e3}), flush=True)
