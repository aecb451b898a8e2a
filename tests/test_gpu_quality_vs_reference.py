"""North-star bar: the approximate path's quality loss (the application's
own metric: MAPE, MCR for K-Means) must match the reference's within 1e-3.
The reference here is the real one — /root/reference's headers compiled into
oracle/_ref — running its own exact and approximate CPU engine with glibc
math, against our CUDA path on the same seeded inputs and grid."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from paper_2308_16877_b200 import abi
from paper_2308_16877_b200 import engine as E
from gpu_util import dev

pytestmark = pytest.mark.gpu

TOL = 1e-3  # north_star: quality loss within 1e-3 of the reference's


def _ref_mape(a, b):
    L = oracle.ref()
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return L.ref_mape(a.ctypes.data, b.ctypes.data, len(a))


@pytest.mark.parametrize("spec_fn", [
    lambda: E.taf(5, 8, 0.5), lambda: E.taf(5, 1, 0.5, "warp"), lambda: E.taf(2, 1, 0.1),
    lambda: E.iact(4, 0.3), lambda: E.iact(4, 0.3, level="warp"), lambda: E.perfo("small", 4),
    lambda: E.perfo("large", 2, level="team")])
def test_blackscholes_quality_matches_reference(spec_fn):
    n = 64 * 64 * 16
    opts = E.make_bs_portfolio(n, 42)
    grid, mp = E.resolve_grid("blackscholes", n)
    ref_exact, ref_apx = np.zeros(n), np.zeros(n)
    assert oracle.ref_run(grid, n, mp, E.blackscholes_region(opts, ref_exact), None)[0] == 0
    assert oracle.ref_run(grid, n, mp, E.blackscholes_region(opts, ref_apx), spec_fn())[0] == 0
    d = dev(opts)
    g_exact = torch.zeros(n, dtype=torch.float64, device="cuda")
    g_apx = torch.zeros(n, dtype=torch.float64, device="cuda")
    E.run_region(grid, n, mp, E.blackscholes_region(d, g_exact), None)
    E.run_region(grid, n, mp, E.blackscholes_region(d, g_apx), spec_fn())
    q_ref, q_gpu = _ref_mape(ref_exact, ref_apx), E.mape(g_exact, g_apx)
    assert abs(q_ref - q_gpu) <= TOL, (q_ref, q_gpu)


@pytest.mark.parametrize("ipt,thr", [(32, 0.5), (32, 2.0)])
def test_binomial_quality_matches_reference(ipt, thr):
    n, steps = 512, 32
    opts = E.make_binomial_portfolio(n, 42)
    grid, mp = E.resolve_grid("binomial", n, items_per_thread=ipt)
    ref_exact, ref_apx = np.zeros(n), np.zeros(n)
    spec = lambda: E.iact(4, thr, level="team")
    assert oracle.ref_run(grid, n, mp, E.binomial_region(opts, steps, ref_exact), None)[0] == 0
    assert oracle.ref_run(grid, n, mp, E.binomial_region(opts, steps, ref_apx), spec())[0] == 0
    d = dev(opts)
    g_exact = torch.zeros(n, dtype=torch.float64, device="cuda")
    g_apx = torch.zeros(n, dtype=torch.float64, device="cuda")
    E.run_region(grid, n, mp, E.binomial_region(d, steps, g_exact), None)
    E.run_region(grid, n, mp, E.binomial_region(d, steps, g_apx), spec())
    q_ref, q_gpu = _ref_mape(ref_exact, ref_apx), E.mape(g_exact, g_apx)
    assert q_ref > 0 and abs(q_ref - q_gpu) <= TOL, (q_ref, q_gpu)


@pytest.mark.parametrize("spec_fn", [lambda: E.perfo("small", 4), lambda: E.perfo("large", 2),
                                     lambda: E.iact(4, 0.0, 1)])
def test_kmeans_lloyd_quality_matches_reference(spec_fn):
    n, d, k = 4096, 8, 16
    pts = E.make_blobs(n, d, k, 5, 30.0)
    grid, _ = E.resolve_grid("kmeans", n)
    L = oracle.ref()

    def ref_run(spec):
        assign = np.zeros(n, np.int32)
        cent = np.zeros((k, d))
        it, conv = C.c_int32(), C.c_int32()
        st = abi.Stats()
        err = C.create_string_buffer(512)
        rc = L.ref_kmeans_benchmark(pts.ctypes.data, n, d, k, C.byref(grid.c()),
                                    C.byref(spec) if spec is not None else None, 40, assign.ctypes.data,
                                    C.byref(it), C.byref(conv), C.byref(st), err, 512)
        assert rc == 0, err.value
        return assign

    ref_e, ref_a = ref_run(None), ref_run(spec_fn())
    gp = dev(pts)
    g_e = E.kmeans_run(grid, gp, k, None, max_iters=40).assignments
    g_a = E.kmeans_run(grid, gp, k, spec_fn(), max_iters=40).assignments
    q_ref = float(np.mean(ref_e != ref_a))
    q_gpu = E.mcr(g_e, g_a)
    assert abs(q_ref - q_gpu) <= TOL, (q_ref, q_gpu)
