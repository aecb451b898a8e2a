"""Generate golden fixtures from the REFERENCE itself (oracle/_ref, the
unmodified simtac headers compiled in this container). Run here, where
/root/reference exists; the .npz files are committed and used by
tests/test_golden.py on any machine (no reference needed there).

  python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))

import oracle  # noqa: E402
from cases import random_case  # noqa: E402
from paper_2308_16877_b200 import abi  # noqa: E402
from paper_2308_16877_b200 import engine as E  # noqa: E402

SPEC_FIELDS = [f for f, _ in abi.Spec._fields_]
STATS = ["total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps",
         "resident_warps", "arena_required", "arena_available", "fail_team", "fail_step", "fail_missing"]


def spec_vec(s):
    return np.array([np.nan if s is None else float(getattr(s, f)) for f in SPEC_FIELDS])


def table_cases():
    rng = np.random.default_rng(20241017)
    out = {}
    for i in range(200):
        c = random_case(rng)
        o = c.init.copy()
        p = np.zeros(c.n, np.uint8)
        rc, st, msg = oracle.ref_run(c.grid, c.n, c.mapping, c.region(o), c.spec, p)
        g = c.grid
        out[f"c{i:03d}"] = dict(
            grid=np.array([g.num_teams, g.threads_per_team, g.warp_size, g.items_per_thread, g.shared_mem_budget_bytes], np.int64),
            meta=np.array([c.n, c.mapping, c.in_dims, c.out_dims, int(c.accumulate), int(c.barrier)], np.int64),
            spec=spec_vec(c.spec), has_spec=np.array([c.spec is not None]),
            inputs=np.zeros((0, 0)) if c.inputs is None else c.inputs, table=c.table,
            encounters=np.zeros(0, np.int32) if c.encounters is None else c.encounters,
            has_enc=np.array([c.encounters is not None]), init=c.init,
            rc=np.array([rc]), stats=np.array([getattr(st, f) for f in STATS], np.int64),
            out=o, paths=p)
    return out


def app_cases():
    """Application-level vectors: reference generators + reference prices."""
    L = oracle.ref()
    import ctypes as C
    bs = np.empty((2048, 5))
    L.ref_make_bs_portfolio(2048, 42, 512, 0.01, bs.ctypes.data)
    bs_price = np.array([_ref_call(L.ref_black_scholes_call, row) for row in bs])
    bino = np.empty((64, 5))
    L.ref_make_binomial_portfolio(64, 42, 0.002, bino.ctypes.data)
    bino_price = {}
    for steps in (16, 128, 1024):
        v = C.c_double()
        bino_price[steps] = np.array([(L.ref_binomial_price(r.ctypes.data, steps, 1, 1, C.byref(v)), v.value)[1] for r in np.ascontiguousarray(bino)])
    blobs = np.empty((1024, 4))
    L.ref_make_blobs(1024, 4, 8, 42, 8.0, blobs.ctypes.data)
    # reference Lloyd loop on blobs (exact and small:4 perforation)
    km = {}
    for name, spec in (("exact", None), ("small4", E.perfo("small", 4))):
        a = np.zeros(1024, np.int32)
        it, cv = C.c_int32(), C.c_int32()
        st = abi.Stats()
        err = C.create_string_buffer(256)
        g = E.GridConfig(4, 64, 32, 4)
        rc = L.ref_kmeans_benchmark(blobs.ctypes.data, 1024, 4, 8, C.byref(g.c()),
                                    C.byref(spec) if spec is not None else None, 40, a.ctypes.data,
                                    C.byref(it), C.byref(cv), C.byref(st), err, 256)
        assert rc == 0
        km[name] = (a, it.value, cv.value, st.total_invocations, st.approx_invocations)
    # TAF traces (taf.hpp / taf_oracle.hpp)
    rng = np.random.default_rng(777)
    traces = []
    for _ in range(64):
        h, p, thr = int(rng.integers(1, 6)), int(rng.integers(1, 9)), float(rng.uniform(0, 0.3))
        stream = np.cumsum(rng.normal(0, 0.02, 120)) + 1.0
        ap = np.zeros(100, np.uint8)
        ov = np.zeros(100)
        m = L.ref_taf_drive(h, p, thr, stream.ctypes.data, len(stream), 100, ap.ctypes.data, ov.ctypes.data)
        traces.append((h, p, thr, stream, ap[:m].copy(), ov[:m].copy()))
    return dict(bs=bs, bs_price=bs_price, bino=bino, bino_price=bino_price, blobs=blobs, km=km, traces=traces)


def _ref_call(f, row):
    import ctypes as C
    v = C.c_double()
    rc = f(np.ascontiguousarray(row).ctypes.data, C.byref(v))
    return v.value if rc == 0 else np.nan


def main():
    tc = table_cases()
    flat = {}
    for key, d in tc.items():
        for f, v in d.items():
            flat[f"{key}/{f}"] = v
    np.savez_compressed(HERE / "engine_table_cases.npz", **flat)
    a = app_cases()
    flat = {"bs": a["bs"], "bs_price": a["bs_price"], "bino": a["bino"], "blobs": a["blobs"]}
    for s, v in a["bino_price"].items():
        flat[f"bino_price_{s}"] = v
    for k, (lab, it, cv, tot, app) in a["km"].items():
        flat[f"km_{k}_labels"] = lab
        flat[f"km_{k}_meta"] = np.array([it, cv, tot, app], np.int64)
    for i, (h, p, thr, stream, ap, ov) in enumerate(a["traces"]):
        flat[f"taf{i:02d}_cfg"] = np.array([h, p, thr])
        flat[f"taf{i:02d}_stream"] = stream
        flat[f"taf{i:02d}_approx"] = ap
        flat[f"taf{i:02d}_out"] = ov
    np.savez_compressed(HERE / "apps.npz", **flat)
    print("wrote", [p.name for p in HERE.glob("*.npz")])


if __name__ == "__main__":
    main()
