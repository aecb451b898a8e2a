"""Blackscholes C1: bs_stream_kernel exact/TAF with one or two logical
threads per CUDA thread (HPAC_STREAM_PAIR), kernel medians."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if len(sys.argv) == 1:
    for pv in ["1", "0"]:  # 1 = paired (opt-in)
        subprocess.run([sys.executable, __file__, pv], env=dict(os.environ, HPAC_STREAM_PAIR=pv))
    sys.exit(0)
import numpy as np, torch
from paper_2308_16877_b200 import engine as E
n = 1 << 22
opts = E.make_bs_portfolio(n, 42)
grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
d = torch.from_numpy(opts).cuda(); o = torch.zeros(n, dtype=torch.float64, device="cuda")
for name, spec in [("exact", None), ("taf(5,1,0.5)", E.taf(5, 1, 0.5)), ("taf warp", E.taf(5, 1, 0.5, level="warp")),
                   ("perfo small:4", E.perfo("small", 4))]:
    ms = [E.run_region(grid, n, mp, E.blackscholes_region(d, o), spec).kernel_ms for _ in range(30)]
    print(f"pair={sys.argv[1]} {name:14s} {np.median(ms)*1e3:7.1f} us", flush=True)
