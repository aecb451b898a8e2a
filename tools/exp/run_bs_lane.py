"""Blackscholes C1: barrier-free lane kernel (default) vs the bulk-TMA tile
kernel (HPAC_STREAM_TMA=1), exact / TAF / perforation, and the iACT engine,
kernel medians (L2 flushed before every launch)."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if len(sys.argv) == 1:
    for tv in ["1", "0"]:
        subprocess.run([sys.executable, __file__, tv], env=dict(os.environ, HPAC_STREAM_TMA=tv))
    sys.exit(0)
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
d = torch.from_numpy(opts).cuda(); o = torch.zeros(n, dtype=torch.float64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for name, spec in [("exact", None), ("taf(5,1,0.5)", E.taf(5, 1, 0.5)), ("taf warp", E.taf(5, 1, 0.5, level="warp")),
                   ("taf team", E.taf(5, 1, 0.5, level="team")), ("perfo small:4", E.perfo("small", 4)),
                   ("iact(2,0.5)", E.iact(2, 0.5)), ("iact(2,0.5) warp", E.iact(2, 0.5, level="warp"))]:
    if sys.argv[1] == "1" and name.startswith("iact"):
        continue
    ms = []
    for _ in range(30):
        flush.fill_(1.0)
        ms.append(E.run_region(grid, n, mp, E.blackscholes_region(d, o), spec).kernel_ms)
    print(f"tma={sys.argv[1]} {name:18s} {np.median(ms)*1e3:7.1f} us", flush=True)
