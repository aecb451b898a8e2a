"""Golden fixtures generated from the reference itself (tests/golden/make_golden.py,
oracle/_ref = /root/reference compiled here). CPU: the oracle and the host
generators must reproduce them bit for bit. GPU: the CUDA engine must too
(tables: bit-exact; application prices: 1e-6 relative)."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import oracle
from cases import Case
from paper_2308_16877_b200 import abi
from paper_2308_16877_b200 import engine as E

G = Path(__file__).resolve().parent / "golden"
SPEC_FIELDS = [f for f, _ in abi.Spec._fields_]
STATS = ["total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps",
         "resident_warps", "arena_required", "arena_available", "fail_team", "fail_step", "fail_missing"]


def _load_cases():
    z = np.load(G / "engine_table_cases.npz")
    keys = sorted({k.split("/")[0] for k in z.files})
    out = []
    for k in keys:
        d = {f.split("/")[1]: z[f] for f in z.files if f.startswith(k + "/")}
        g = d["grid"]
        n, mapping, in_dims, out_dims, acc, bar = (int(x) for x in d["meta"])
        spec = None
        if d["has_spec"][0]:
            spec = abi.Spec()
            for f, v in zip(SPEC_FIELDS, d["spec"]):
                ctype = dict(abi.Spec._fields_)[f]
                setattr(spec, f, float(v) if ctype is C.c_double else int(v))
        case = Case(E.GridConfig(int(g[0]), int(g[1]), int(g[2]), int(g[3]), int(g[4])), n, mapping,
                    in_dims, out_dims, d["inputs"] if in_dims > 0 else None, d["table"],
                    d["encounters"] if d["has_enc"][0] else None, bool(acc), bool(bar), spec, d["init"])
        out.append((k, case, int(d["rc"][0]), d["stats"], d["out"], d["paths"]))
    return out


CASES = _load_cases()


def _check(rc, st_vec, out, paths, case, exp_rc, exp_st, exp_out, exp_paths, key, abort_outputs=True):
    assert rc == exp_rc, key
    exp = dict(zip(STATS, exp_st))
    if rc == 0:
        for f in STATS[:5]:
            assert st_vec[f] == exp[f], (key, f)
        assert np.array_equal(paths, exp_paths), key
    if rc == 0 or (rc == 3 and abort_outputs):
        # (on BarrierDivergenceError the reference aborts mid-run; the device
        # reports the same error but outputs after the abort are unspecified)
        assert np.array_equal(out, exp_out), key
    if rc == 2:
        assert (st_vec["arena_required"], st_vec["arena_available"]) == (exp["arena_required"], exp["arena_available"]), key
    if rc == 3:
        assert (st_vec["fail_team"], st_vec["fail_step"], st_vec["fail_missing"]) == \
            (exp["fail_team"], exp["fail_step"], exp["fail_missing"]), key


def test_oracle_reproduces_reference_table_fixtures():
    assert len(CASES) == 200
    for key, case, exp_rc, exp_st, exp_out, exp_paths in CASES:
        o = case.init.copy()
        p = np.zeros(case.n, np.uint8)
        rc, st, msg = oracle.oracle_run(case.grid, case.n, case.mapping, case.region(o), case.spec, p)
        _check(rc, {f: getattr(st, f) for f in STATS}, o, p, case, exp_rc, exp_st, exp_out, exp_paths, key)


@pytest.mark.gpu
def test_cuda_reproduces_reference_table_fixtures():
    from gpu_util import run_case_gpu
    for key, case, exp_rc, exp_st, exp_out, exp_paths in CASES:
        rc, st, out, paths, msg = run_case_gpu(case)
        full = {f: st.get(f, 0) for f in STATS}
        _check(rc, full, out, paths, case, exp_rc, exp_st, exp_out, exp_paths, key + " " + msg,
               abort_outputs=False)


APPS = np.load(G / "apps.npz")


def test_generators_reproduce_reference_fixtures():
    assert np.array_equal(E.make_bs_portfolio(2048, 42), APPS["bs"])
    assert np.array_equal(E.make_binomial_portfolio(64, 42), APPS["bino"])
    assert np.array_equal(E.make_blobs(1024, 4, 8, 42, 8.0), APPS["blobs"])


def test_oracle_prices_match_reference_fixtures():
    assert np.array_equal(oracle.bs_prices(APPS["bs"]), APPS["bs_price"])
    for steps in (16, 128, 1024):
        assert np.array_equal(oracle.binomial_prices(APPS["bino"], steps), APPS[f"bino_price_{steps}"])


def test_oracle_taf_traces_match_reference():
    L = oracle.oracle()
    for i in range(64):
        h, p, thr = APPS[f"taf{i:02d}_cfg"]
        s = APPS[f"taf{i:02d}_stream"]
        ap = np.zeros(100, np.uint8)
        ov = np.zeros(100)
        m = L.oracle_taf_drive(int(h), int(p), float(thr), s.ctypes.data, len(s), 100, ap.ctypes.data, ov.ctypes.data)
        assert np.array_equal(ap[:m], APPS[f"taf{i:02d}_approx"])
        assert np.array_equal(ov[:m], APPS[f"taf{i:02d}_out"])


def test_oracle_kmeans_matches_reference_fixture():
    pts = APPS["blobs"]
    for name, spec in (("exact", None), ("small4", E.perfo("small", 4))):
        a = np.zeros(1024, np.int32)
        it, cv = C.c_int32(), C.c_int32()
        st = abi.Stats()
        err = C.create_string_buffer(256)
        g = E.GridConfig(4, 64, 32, 4)
        rc = oracle.oracle().oracle_kmeans_benchmark(pts.ctypes.data, 1024, 4, 8, C.byref(g.c()),
                                                     C.byref(spec) if spec is not None else None, 40, 0,
                                                     a.ctypes.data, None, C.byref(it), C.byref(cv),
                                                     C.byref(st), err, 256)
        assert rc == 0
        meta = APPS[f"km_{name}_meta"]
        assert [it.value, cv.value, st.total_invocations, st.approx_invocations] == list(meta)
        assert np.array_equal(a, APPS[f"km_{name}_labels"])


@pytest.mark.gpu
def test_cuda_prices_match_reference_fixtures():
    import torch
    bs = APPS["bs"]
    out = torch.zeros(len(bs), dtype=torch.float64, device="cuda")
    E.run_region(E.GridConfig(2, 64, 32, 16), len(bs), 0, E.blackscholes_region(torch.from_numpy(bs).cuda(), out), None)
    want = APPS["bs_price"]
    assert np.all(np.abs(out.cpu().numpy() - want) <= 1e-6 * np.abs(want))
    bino = APPS["bino"]
    for steps in (16, 128, 1024):
        o = torch.zeros(len(bino), dtype=torch.float64, device="cuda")
        E.run_region(E.GridConfig(len(bino), 64, 32, 1), len(bino), 1,
                     E.binomial_region(torch.from_numpy(bino).cuda(), steps, o), None)
        w = APPS[f"bino_price_{steps}"]
        assert np.all(np.abs(o.cpu().numpy() - w) <= 1e-6 * np.abs(w)), steps


@pytest.mark.gpu
def test_cuda_kmeans_matches_reference_fixture():
    import torch
    pts = torch.from_numpy(APPS["blobs"]).cuda()
    for name, spec in (("exact", None), ("small4", E.perfo("small", 4))):
        r = E.kmeans_run(E.GridConfig(4, 64, 32, 4), pts, 8, spec)
        meta = APPS[f"km_{name}_meta"]
        assert [r.iterations, int(r.converged), r.stats["total_invocations"], r.stats["approx_invocations"]] == list(meta)
        mcr = float(np.mean(r.assignments.cpu().numpy() != APPS[f"km_{name}_labels"]))
        assert mcr <= 1e-3
