"""Quality map of TAF on LavaMD (C4) on the CPU oracle: approximation rate and
MAPE of fv vs the exact run, per (level, h, p, thr). Small box grid so the
oracle finishes quickly; prints one JSON line per point."""
import itertools
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2308_16877_b200 import engine as E  # noqa: E402

B1 = int(os.environ.get("B1", 6))
P = int(os.environ.get("P", 128))
IPT = int(os.environ.get("IPT", 1))


def run(spec_args):
    rv, qv = E.make_lavamd(B1, P, 42)
    nb = B1 ** 3
    grid = E.GridConfig((nb + IPT - 1) // IPT, P, 32, IPT)
    fv = np.zeros((nb * P, 4))
    spec = None if spec_args is None else E.taf(*spec_args)
    rc, st, msg = oracle.oracle_run(grid, nb, 1, E.lavamd_region(rv, qv, fv, B1, P), spec)
    assert rc == 0, msg
    return fv, st.approx_invocations / max(1, st.total_invocations), st.divergent_warp_steps / max(1, st.total_warp_steps)


def point(args):
    fv, rate, div = run(args)
    return args, rate, div, fv


if __name__ == "__main__":
    exact, _, _ = run(None)
    levels = sys.argv[1].split(",") if len(sys.argv) > 1 else ["thread", "warp", "team"]
    pts = [(h, p, thr, lv) for lv in levels for h in (1, 2, 3) for p in (1, 2, 4, 8)
           for thr in (0.02, 0.05, 0.1, 0.2, 0.5)]
    with ProcessPoolExecutor(os.cpu_count()) as ex:
        for args, rate, div, fv in ex.map(point, pts):
            d = np.abs(fv - exact)
            mape = float(np.mean(d / np.abs(exact)))
            mape_v = float(np.mean(d[:, 0] / np.abs(exact[:, 0])))
            rel_l2 = float(np.linalg.norm(fv - exact) / np.linalg.norm(exact))
            print(json.dumps({"h": args[0], "p": args[1], "thr": args[2], "level": args[3],
                              "rate": round(rate, 4), "mape": round(mape, 5), "mape_v": round(mape_v, 5),
                              "rel_l2": round(rel_l2, 5), "div": round(div, 4)}), flush=True)
