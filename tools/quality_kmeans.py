"""Quality map of the K-Means Lloyd loop (bench/kmeans.hpp:62-144) under
perforation on the CPU oracle: final-label MCR vs the exact run with the
same iteration budget, skip rate, iterations. Prints one JSON line per point."""
import ctypes as C
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2308_16877_b200 import abi  # noqa: E402
from paper_2308_16877_b200 import engine as E  # noqa: E402

N = int(os.environ.get("N", 1 << 16))
D, K = 32, 64
SEP = float(os.environ.get("SEP", 8.0))
ITERS = int(os.environ.get("ITERS", 40))


def run(spec_args, ipt=4):
    pts = E.make_blobs(N, D, K, 42, SEP)
    grid, _ = E.resolve_grid("kmeans", N, items_per_thread=ipt)
    spec = None
    if spec_args is not None:
        spec = E.perfo(spec_args[0], spec_args[1], level=spec_args[2] if len(spec_args) > 2 else "thread", seed=0)
    assign = np.zeros(N, np.int32)
    cent = np.zeros((K, D))
    st = abi.Stats()
    err = C.create_string_buffer(512)
    it, conv = C.c_int32(), C.c_int32()
    rc = oracle.oracle().oracle_kmeans_benchmark(pts.ctypes.data, N, D, K, C.byref(grid.c()),
                                                 C.byref(spec) if spec is not None else None, ITERS, 7,
                                                 assign.ctypes.data, cent.ctypes.data, C.byref(it),
                                                 C.byref(conv), C.byref(st), err, 512)
    assert rc == 0, err.value
    return assign, it.value, bool(conv.value), st.approx_invocations / max(1, st.total_invocations)


def point(a):
    return a, run(a)


if __name__ == "__main__":
    exact, it_e, conv_e, _ = run(None)
    print(json.dumps({"spec": None, "iterations": it_e, "converged": conv_e}), flush=True)
    pts = [("random", p, lv) for lv in ("thread", "warp") for p in (10, 25, 50, 75)] + \
        [("small", 2), ("small", 4), ("large", 2)]
    with ProcessPoolExecutor(min(8, os.cpu_count())) as ex:
        for a, (lab, it, conv, rate) in ex.map(point, pts):
            print(json.dumps({"spec": a, "mcr": float(np.mean(lab != exact)), "skip_rate": round(rate, 4),
                              "iterations": it, "converged": conv}), flush=True)
