"""Application regions on the GPU vs the oracle.

* Exact paths: GPU outputs vs the CPU restatement within 1e-6 relative
  (north_star tolerance; CUDA vs glibc libm differ by ulps).
* Approximate paths: decisions depend on output values (TAF) or inputs
  (iACT, perforation). The oracle replays the GPU's own exact outputs
  through the reference engine semantics, so decisions,
  stats, paths and approximated outputs must match bit for bit.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2308_16877_b200 import abi
from paper_2308_16877_b200 import engine as E
from gpu_util import dev

pytestmark = pytest.mark.gpu

REL = 1e-6  # north_star: exact-path outputs within 1e-6 relative
STAT_FIELDS = ["total_invocations", "approx_invocations", "divergent_warp_steps",
               "total_warp_steps", "resident_warps"]


def _rel_ok(got, want, rel=REL):
    got = np.asarray(got)
    want = np.asarray(want)
    return np.all(np.abs(got - want) <= rel * np.abs(want) + 1e-300), \
        float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


def _replay(grid, n, mapping, inputs, exact, spec, init=None):
    out = np.zeros(n) if init is None else init.copy()
    paths = np.zeros(n, np.uint8)
    reg = E.table_region(inputs, exact.reshape(n, 1), out)
    rc, st, msg = oracle.oracle_run(grid, n, mapping, reg, spec, paths)
    assert rc == 0, msg
    return st, out, paths


def _gpu_run(grid, n, mapping, region_fn, spec):
    out = torch.zeros(n, dtype=torch.float64, device="cuda")
    paths = torch.zeros(n, dtype=torch.uint8, device="cuda")
    lr = E.run_region(grid, n, mapping, region_fn(out), spec, paths=paths)
    return lr, out.cpu().numpy(), paths.cpu().numpy()


def _compare(lr, st, g_out, o_out, g_paths, o_paths):
    for f in STAT_FIELDS:
        assert lr.stats[f] == getattr(st, f), f
    assert np.array_equal(g_paths, o_paths)
    assert np.array_equal(g_out, o_out)


# ---------------------------------------------------------------- Black-Scholes

@pytest.fixture(scope="module")
def bs_case():
    n = 64 * 256 * 16  # 256 teams x 64 threads x ipt 16 (C1 shape, 1/16 size)
    opts = E.make_bs_portfolio(n, 42)
    grid, mapping = E.resolve_grid("blackscholes", n)
    d_opts = dev(opts)
    lr, exact, _ = _gpu_run(grid, n, mapping, lambda o: E.blackscholes_region(d_opts, o), None)
    return n, opts, d_opts, grid, mapping, exact, lr


def test_bs_exact_matches_cpu(bs_case):
    n, opts, _, _, _, exact, lr = bs_case
    want = oracle.bs_prices(opts)
    ok, worst = _rel_ok(exact, want)
    assert ok, worst
    assert lr.stats["total_invocations"] == n and lr.stats["approx_invocations"] == 0


def test_bs_atm_reference_value():
    o = np.array([[100.0, 100.0, 0.05, 0.2, 1.0], [100.0, 80.0, 0.05, 0.0, 1.0],
                  [50.0, 80.0, 0.05, 0.0, 1.0]])
    g = E.GridConfig(1, 32, 32, 1)
    lr, out, _ = _gpu_run(g, 3, 0, lambda p: E.blackscholes_region(dev(o), p), None)
    assert abs(out[0] - 10.4506) < 5e-5  # test_bench.cpp:50-53
    assert abs(out[1] - (100.0 - 80.0 * np.exp(-0.05))) < 1e-12  # test_bench.cpp:60-63
    assert out[2] == 0.0


def test_bs_invalid_parameters_raise():
    o = np.array([[-1.0, 100.0, 0.05, 0.2, 1.0]])
    g = E.GridConfig(1, 32, 32, 1)
    with pytest.raises(E.ConfigError):
        _gpu_run(g, 1, 0, lambda p: E.blackscholes_region(dev(o), p), None)


@pytest.mark.parametrize("level", ["thread", "warp", "team"])
@pytest.mark.parametrize("spec_args", [(5, 1, 0.5), (5, 8, 0.5), (2, 8, float("inf")), (3, 4, 0.05), (12, 3, 0.5)])
def test_bs_taf_decisions_bit_exact(bs_case, level, spec_args):
    n, opts, d_opts, grid, mapping, exact, _ = bs_case
    spec = E.taf(*spec_args, level=level)
    lr, g_out, g_paths = _gpu_run(grid, n, mapping, lambda o: E.blackscholes_region(d_opts, o), spec)
    st, o_out, o_paths = _replay(grid, n, mapping, opts, exact, E.taf(*spec_args, level=level))
    _compare(lr, st, g_out, o_out, g_paths, o_paths)


@pytest.mark.parametrize("args", [(2, 0.5, None, "thread"), (4, 0.3, None, "thread"),
                                  (8, 0.3, None, "thread"), (4, 0.3, None, "warp"),
                                  (2, 0.5, 4, "thread"), (3, 0.5, 1, "team")])
def test_bs_iact_decisions_bit_exact(bs_case, args):
    n, opts, d_opts, grid, mapping, exact, _ = bs_case
    sub = 64 * 64 * 16  # keep the oracle quick
    spec = E.iact(args[0], args[1], args[2], args[3])
    g = E.GridConfig(64, 64, 32, 16)
    lr, g_out, g_paths = _gpu_run(g, sub, mapping, lambda o: E.blackscholes_region(d_opts[:sub], o), spec)
    st, o_out, o_paths = _replay(g, sub, mapping, opts[:sub], exact[:sub], E.iact(args[0], args[1], args[2], args[3]))
    _compare(lr, st, g_out, o_out, g_paths, o_paths)


@pytest.mark.parametrize("kind,arg", [("small", 4), ("large", 2), ("ini", 25), ("fini", 10),
                                      ("herded_small", 4), ("random", 30)])
def test_bs_perfo_bit_exact(bs_case, kind, arg):
    n, opts, d_opts, grid, mapping, exact, _ = bs_case
    spec = E.perfo(kind, arg, seed=123)
    lr, g_out, g_paths = _gpu_run(grid, n, mapping, lambda o: E.blackscholes_region(d_opts, o), spec)
    st, o_out, o_paths = _replay(grid, n, mapping, opts, exact, E.perfo(kind, arg, seed=123))
    _compare(lr, st, g_out, o_out, g_paths, o_paths)


# ---------------------------------------------------------------- Binomial

@pytest.mark.parametrize("steps", [1, 2, 16, 31, 32, 33, 100, 1023, 1024, 1055, 1056, 1500])
def test_binomial_exact_matches_cpu(steps):
    n = 48
    opts = E.make_binomial_portfolio(n, 7)
    grid = E.GridConfig(n, 64, 32, 1)
    lr, out, _ = _gpu_run(grid, n, 1, lambda o: E.binomial_region(dev(opts), steps, o), None)
    want = oracle.binomial_prices(opts, steps)
    ok, worst = _rel_ok(out, want)
    assert ok, (steps, worst)
    assert lr.stats["total_invocations"] == n * 64
    assert lr.stats["total_warp_steps"] == n * 2


@pytest.mark.parametrize("american,put", [(True, True), (False, True), (True, False), (False, False)])
def test_binomial_variants(american, put):
    n = 16
    opts = E.make_binomial_portfolio(n, 3)
    grid = E.GridConfig(n, 64, 32, 1)
    lr, out, _ = _gpu_run(grid, n, 1, lambda o: E.binomial_region(dev(opts), 256, o, american, put), None)
    want = oracle.binomial_prices(opts, 256, american, put)
    ok, worst = _rel_ok(out, want)
    assert ok, worst


def test_binomial_one_step_by_hand():
    o = np.array([[100.0, 105.0, 0.05, 0.3, 1.0]])
    u = np.exp(0.3)
    d = 1 / u
    g = np.exp(0.05)
    p = (g - d) / (u - d)
    cont = (p * max(105 - 100 * u, 0) + (1 - p) * max(105 - 100 * d, 0)) / g
    want = max(cont, 105 - 100.0)  # test_bench.cpp:36-46
    lr, out, _ = _gpu_run(E.GridConfig(1, 64, 32, 1), 1, 1, lambda p_: E.binomial_region(dev(o), 1, p_), None)
    assert abs(out[0] - want) <= 1e-15 * want * 8


@pytest.mark.parametrize("ipt,thr,tsize", [(8, 0.5, 4), (64, 0.5, 4), (64, 2.0, 4), (128, 0.5, 8), (300, 0.5, 2),
                                            (64, 0.5, 3), (64, 1.0, 5), (64, 0.3, 7), (128, 0.5, 12)])
def test_binomial_iact_team_decisions_bit_exact(ipt, thr, tsize):
    steps = 64
    n = 96 * ipt
    opts = E.make_binomial_portfolio(n, 42)
    grid, mapping = E.resolve_grid("binomial", n, items_per_thread=ipt)
    d_opts = dev(opts)
    _, exact, _ = _gpu_run(grid, n, mapping, lambda o: E.binomial_region(d_opts, steps, o), None)
    spec = E.iact(tsize, thr, level="team")
    lr, g_out, g_paths = _gpu_run(grid, n, mapping, lambda o: E.binomial_region(d_opts, steps, o), spec)
    st, o_out, o_paths = _replay(grid, n, mapping, opts, exact, E.iact(tsize, thr, level="team"))
    _compare(lr, st, g_out, o_out, g_paths, o_paths)
    assert lr.stats["divergent_warp_steps"] == 0


def test_binomial_duplicates_zero_error():
    """test_bench.cpp:95-126: warm team tables on duplicated options."""
    opts = np.array([[100.0, 90.0 + 10.0 * k, 0.05, 0.25, 1.0] for rep in range(8) for k in range(4)])
    n = len(opts)
    grid = E.GridConfig(4, 32, 32, n // 4)
    d = dev(opts)
    _, acc, _ = _gpu_run(grid, n, 1, lambda o: E.binomial_region(d, 16, o), None)
    lr, app, _ = _gpu_run(grid, n, 1, lambda o: E.binomial_region(d, 16, o), E.iact(4, 0.0))
    assert lr.approx_rate() > 0.0
    assert oracle.oracle().oracle_mape(acc.ctypes.data, app.ctypes.data, n) == 0.0


@pytest.mark.parametrize("kind,arg", [("small", 4), ("large", 4), ("ini", 10), ("random", 25)])
def test_binomial_perfo_bit_exact(kind, arg):
    steps, ipt = 32, 16
    n = 50 * ipt
    opts = E.make_binomial_portfolio(n, 5)
    grid, mapping = E.resolve_grid("binomial", n, items_per_thread=ipt)
    d_opts = dev(opts)
    _, exact, _ = _gpu_run(grid, n, mapping, lambda o: E.binomial_region(d_opts, steps, o), None)
    lr, g_out, g_paths = _gpu_run(grid, n, mapping, lambda o: E.binomial_region(d_opts, steps, o), E.perfo(kind, arg, seed=9))
    st, o_out, o_paths = _replay(grid, n, mapping, opts, exact, E.perfo(kind, arg, seed=9))
    _compare(lr, st, g_out, o_out, g_paths, o_paths)


@pytest.mark.parametrize("h,p,thr", [(2, 4, 0.01), (1, 8, 0.5), (3, 2, float("inf"))])
def test_binomial_taf_bit_exact(h, p, thr):
    steps, ipt = 32, 24
    n = 20 * ipt
    opts = E.make_binomial_portfolio(n, 11)
    grid, mapping = E.resolve_grid("binomial", n, items_per_thread=ipt)
    d_opts = dev(opts)
    _, exact, _ = _gpu_run(grid, n, mapping, lambda o: E.binomial_region(d_opts, steps, o), None)
    lr, g_out, g_paths = _gpu_run(grid, n, mapping, lambda o: E.binomial_region(d_opts, steps, o), E.taf(h, p, thr, "team"))
    st, o_out, o_paths = _replay(grid, n, mapping, opts, exact, E.taf(h, p, thr, "team"))
    _compare(lr, st, g_out, o_out, g_paths, o_paths)


# ---------------------------------------------------------------- K-Means region

def _km_oracle(points, cents, spec, grid, n):
    labels = np.zeros(n, np.int32)
    dist = np.zeros((n, cents.shape[0]))
    paths = np.zeros(n, np.uint8)
    reg = E.kmeans_region(points, cents, labels, dist)
    rc, st, msg = oracle.oracle_run(grid, n, 0, reg, spec, paths)
    assert rc == 0, msg
    return st, labels, dist, paths


@pytest.mark.parametrize("spec_fn", [lambda: None, lambda: E.perfo("small", 2), lambda: E.perfo("large", 4),
                                     lambda: E.perfo("random", 30, seed=5), lambda: E.iact(2, 0.0, 1),
                                     lambda: E.perfo("herded_small", 3, level="warp")])
def test_kmeans_region_labels_bit_exact(spec_fn):
    n, d, k = 64 * 32 * 4, 32, 64
    pts = E.make_blobs(n, d, k, 42, 8.0)
    rng = np.random.default_rng(1)
    cents = pts[rng.choice(n, k, replace=False)].copy()
    grid, _ = E.resolve_grid("kmeans", n)
    labels = torch.zeros(n, dtype=torch.int32, device="cuda")
    paths = torch.zeros(n, dtype=torch.uint8, device="cuda")
    spec = spec_fn()
    lr = E.run_region(grid, n, 0, E.kmeans_region(dev(pts), dev(cents), labels), spec, paths=paths)
    st, o_labels, _, o_paths = _km_oracle(pts, cents, spec_fn(), grid, n)
    for f in STAT_FIELDS:
        assert lr.stats[f] == getattr(st, f), f
    assert np.array_equal(paths.cpu().numpy(), o_paths)
    assert np.array_equal(labels.cpu().numpy(), o_labels)


def test_kmeans_distances_output_exact():
    n, d, k = 2048, 8, 16
    pts = E.make_blobs(n, d, k, 3, 8.0)
    cents = pts[:k].copy()
    grid, _ = E.resolve_grid("kmeans", n)
    labels = torch.zeros(n, dtype=torch.int32, device="cuda")
    dist = torch.zeros((n, k), dtype=torch.float64, device="cuda")
    E.run_region(grid, n, 0, E.kmeans_region(dev(pts), dev(cents), labels, dist), None)
    _, o_labels, o_dist, _ = _km_oracle(pts, cents, None, grid, n)
    assert np.array_equal(dist.cpu().numpy(), o_dist)
    assert np.array_equal(labels.cpu().numpy(), o_labels)


# ---------------------------------------------------------------- synthetic

@pytest.mark.parametrize("profile", [0, 1, 2])
@pytest.mark.parametrize("spec_fn", [lambda: None, lambda: E.taf(2, 8, float("inf")), lambda: E.taf(2, 16, 0.01, "warp"),
                                     lambda: E.iact(2, 0.5), lambda: E.perfo("small", 4)])
def test_synthetic_bit_exact(profile, spec_fn):
    n = 16384
    grid, mapping = E.resolve_grid("synthetic-constant", n)
    out = torch.zeros(n, dtype=torch.float64, device="cuda")
    paths = torch.zeros(n, dtype=torch.uint8, device="cuda")
    lr = E.run_region(grid, n, mapping, E.synthetic_region(profile, 99, out), spec_fn(), paths=paths)
    o_out = np.zeros(n)
    o_paths = np.zeros(n, np.uint8)
    rc, st, msg = oracle.oracle_run(grid, n, mapping, E.synthetic_region(profile, 99, o_out), spec_fn(), o_paths)
    assert rc == 0, msg
    _compare(lr, st, out.cpu().numpy(), o_out, paths.cpu().numpy(), o_paths)


@pytest.mark.parametrize("steps", [16, 40, 64, 96, 128, 200, 256, 512, 1000])
def test_binomial_american_put_grid_of_moneyness(steps):
    """The American-put lattice skips the exercise region below a tracked
    bound and the exactly-zero region above the highest in-the-money leaf;
    sweep moneyness / volatility / maturity so both edges land everywhere in
    the lane blocks (incl. the block's top node being the zero node)."""
    rng = np.random.default_rng(steps)
    m = 192
    S = 100.0 * np.ones(m)
    K = S * np.exp(rng.uniform(np.log(0.6), np.log(1.6), m))
    r = rng.uniform(0.0, 0.08, m)
    vol = rng.uniform(0.05, 0.8, m)
    T = rng.uniform(0.1, 3.0, m)
    opts = np.stack([S, K, r, vol, T], 1)
    want = oracle.binomial_prices(opts, steps)
    out = torch.zeros(m, dtype=torch.float64, device="cuda")
    lr = E.run_region(E.GridConfig(m, 64, 32, 1), m, 1, E.binomial_region(dev(opts), steps, out), None)
    ok, worst = _rel_ok(out.cpu().numpy(), want)
    assert ok, worst


@pytest.mark.parametrize("tsize", [16, 32, 40])
def test_binomial_iact_large_tables_bit_exact(tsize):
    # tables past the default 48 KiB arena (a larger shared_mem_budget):
    # the decide kernel's lane-per-slot table up to 32 slots, the lane-0
    # scan beyond
    steps, ipt = 64, 64
    n = 64 * ipt
    opts = E.make_binomial_portfolio(n, 43)
    grid, mapping = E.resolve_grid("binomial", n, items_per_thread=ipt)
    grid.shared_mem_budget_bytes = 200 * 1024
    d_opts = dev(opts)
    _, exact, _ = _gpu_run(grid, n, mapping, lambda o: E.binomial_region(d_opts, steps, o), None)
    spec = E.iact(tsize, 0.5, level="team")
    lr, g_out, g_paths = _gpu_run(grid, n, mapping, lambda o: E.binomial_region(d_opts, steps, o), spec)
    st, o_out, o_paths = _replay(grid, n, mapping, opts, exact, E.iact(tsize, 0.5, level="team"))
    _compare(lr, st, g_out, o_out, g_paths, o_paths)
