"""Blackscholes C1: thread-level TAF / perforation, lane-asynchronous kernel
(default) vs lockstep lane kernel (HPAC_STREAM_ASYNC=0); kernel medians, L2 flushed."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if len(sys.argv) == 1:
    for av in ["0", "1"]:
        subprocess.run([sys.executable, __file__, av], env=dict(os.environ, HPAC_STREAM_ASYNC=av))
    sys.exit(0)
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
d = torch.from_numpy(opts).cuda(); o = torch.zeros(n, dtype=torch.float64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for name, spec in [("exact", None), ("taf(5,1,0.5)", E.taf(5, 1, 0.5)), ("taf(5,8,0.5)", E.taf(5, 8, 0.5)),
                   ("taf(2,8,0.5)", E.taf(2, 8, 0.5)), ("perfo small:4", E.perfo("small", 4)),
                   ("perfo random:25", E.perfo("random", 25)), ("perfo random:50", E.perfo("random", 50))]:
    ms = []
    for _ in range(30):
        flush.fill_(1.0)
        lr = E.run_region(grid, n, mp, E.blackscholes_region(d, o), spec)
        ms.append(lr.kernel_ms)
    print(f"async={sys.argv[1]} {name:16s} {np.median(ms)*1e3:7.1f} us  approx {lr.approx_rate():.3f}", flush=True)
