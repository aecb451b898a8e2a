"""The streaming per-thread engines (csrc/engine_stream.cu: barrier-free lane
kernel and bulk-TMA staged input tiles; csrc/engine_bs_iact.cu: iACT decide-then-price) against the generic per-thread engine (HPAC_ENGINE=thread) and
the oracle, on ragged shapes the C1 grid never exercises: partial last
tiles (per-thread fallback loads), logical warps narrower than 32, teams of
32..256 threads, every decision level, TAF and perforation."""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2308_16877_b200 import engine as E
from gpu_util import dev

pytestmark = pytest.mark.gpu

STAT_FIELDS = ["total_invocations", "approx_invocations", "divergent_warp_steps",
               "total_warp_steps", "resident_warps"]


def _run(grid, n, d_opts, spec_fn, engine=None):
    out = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
    paths = torch.zeros(n, dtype=torch.uint8, device="cuda")
    old = os.environ.pop("HPAC_ENGINE", None)
    if engine:
        os.environ["HPAC_ENGINE"] = engine
    try:
        lr = E.run_region(grid, n, 0, E.blackscholes_region(d_opts, out), spec_fn(), paths=paths)
    finally:
        os.environ.pop("HPAC_ENGINE", None)
        if old is not None:
            os.environ["HPAC_ENGINE"] = old
    return lr, out.cpu().numpy(), paths.cpu().numpy()


SHAPES = [  # (num_teams, tpt, ws, ipt, n)
    (37, 64, 32, 5, 37 * 64 * 5 - 17),
    (16, 32, 8, 7, 16 * 32 * 7 - 1),
    (9, 128, 16, 4, 9 * 128 * 3 + 65),
    (5, 256, 32, 3, 5 * 256 * 3 - 300),
    (64, 64, 4, 16, 64 * 64 * 16),
    (1024, 64, 32, 16, 1024 * 64 * 16),  # C1 shape at 1/4 size
]
SPECS = [
    lambda: None,
    lambda: E.taf(5, 1, 0.5, "thread"),
    lambda: E.taf(3, 4, 0.05, "warp"),
    lambda: E.taf(2, 8, float("inf"), "team"),
    lambda: E.taf(8, 2, 0.3, "thread"),
    lambda: E.perfo("small", 3),
    lambda: E.perfo("large", 2, level="warp"),
    lambda: E.perfo("fini", 30),
    lambda: E.perfo("random", 40, seed=9, level="team"),
    lambda: E.perfo("herded_large", 3),
    # approximate steps where no lane waits on a prefetched tile (the buffer
    # is re-armed two steps later: the engine must retire the old copy first)
    lambda: E.taf(5, 2, 0.1, "warp"),
    lambda: E.taf(5, 8, 0.5, "team"),
    lambda: E.taf(2, 1, 1.0, "warp"),
    # iACT: the decide-then-price engine (engine_bs_iact.cu)
    lambda: E.iact(2, 0.5),
    lambda: E.iact(4, 0.3, 2, "warp"),
    lambda: E.iact(3, 0.5, 1, "team"),
    lambda: E.iact(8, 0.2),
    lambda: E.iact(1, float("inf"), 1, "warp"),
    lambda: E.iact(4, 0.0, None, "team"),
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("si", range(len(SPECS)))
def test_stream_engine_equals_generic_engine(shape, si):
    teams, tpt, ws, ipt, n = shape
    opts = E.make_bs_portfolio(n, 11)
    d_opts = dev(opts)
    grid = E.GridConfig(teams, tpt, ws, ipt)
    try:
        a = _run(grid, n, d_opts, SPECS[si])
    except E.ArenaOverflowError as e:
        # the reference's arena charge (bind_technique) applies to both engines
        with pytest.raises(E.ArenaOverflowError) as f:
            _run(grid, n, d_opts, SPECS[si], engine="thread")
        assert (e.required_bytes, e.available_bytes) == (f.value.required_bytes,
                                                         f.value.available_bytes)
        return
    b = _run(grid, n, d_opts, SPECS[si], engine="thread")
    for f in STAT_FIELDS:
        assert a[0].stats[f] == b[0].stats[f], f
    assert np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])


@pytest.mark.parametrize("si", [1, 2, 3, 6, 8, 13, 14, 15])
def test_stream_engine_vs_oracle_ragged(si):
    teams, tpt, ws, ipt, n = SHAPES[0]
    opts = E.make_bs_portfolio(n, 5)
    d_opts = dev(opts)
    grid = E.GridConfig(teams, tpt, ws, ipt)
    _, exact, _ = _run(grid, n, d_opts, lambda: None)
    lr, g_out, g_paths = _run(grid, n, d_opts, SPECS[si])
    o_out = np.full(n, -1.0)
    o_paths = np.zeros(n, np.uint8)
    rc, st, msg = oracle.oracle_run(grid, n, 0, E.table_region(opts, exact.reshape(n, 1), o_out),
                                    SPECS[si](), o_paths)
    assert rc == 0, msg
    for f in STAT_FIELDS:
        assert lr.stats[f] == getattr(st, f), f
    assert np.array_equal(g_paths, o_paths)
    assert np.array_equal(g_out, o_out)


@pytest.mark.parametrize("tma", ["0", "1"])
def test_stream_engine_misaligned_input_falls_back(tma, monkeypatch):
    # a view starting 8 bytes into the buffer defeats the 16-byte bulk-copy
    # alignment; the tile kernel must take per-thread loads and stay exact
    monkeypatch.setenv("HPAC_STREAM_TMA", tma)
    n = 32 * 64 * 4
    opts = E.make_bs_portfolio(n + 1, 3)
    buf = torch.from_numpy(np.concatenate([[0.0], opts.reshape(-1)])).cuda()
    d_view = buf[1:].view(n + 1, 5)[:n]
    grid = E.GridConfig(32, 64, 32, 4)
    a = _run(grid, n, d_view, lambda: E.taf(5, 1, 0.5))
    b = _run(grid, n, dev(opts[:n]), lambda: E.taf(5, 1, 0.5))
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_iact_engine_misaligned_input_falls_back():
    n = 32 * 64 * 4
    opts = E.make_bs_portfolio(n + 1, 3)
    buf = torch.from_numpy(np.concatenate([[0.0], opts.reshape(-1)])).cuda()
    d_view = buf[1:].view(n + 1, 5)[:n]
    grid = E.GridConfig(32, 64, 32, 4)
    a = _run(grid, n, d_view, lambda: E.iact(2, 0.5))
    b = _run(grid, n, dev(opts[:n]), lambda: E.iact(2, 0.5))
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_iact_engine_without_output_buffer():
    # out = NULL: decisions and stats only (the hit copies have no target)
    n = 16 * 64 * 8
    opts = E.make_bs_portfolio(n, 4)
    grid = E.GridConfig(16, 64, 32, 8)
    lr = E.run_region(grid, n, 0, E.blackscholes_region(dev(opts), None), E.iact(2, 0.5))
    ref = _run(grid, n, dev(opts), lambda: E.iact(2, 0.5), engine="thread")[0]
    for f in STAT_FIELDS:
        assert lr.stats[f] == ref.stats[f], f


@pytest.mark.parametrize("shape", [SHAPES[0], SHAPES[3], SHAPES[4]])
@pytest.mark.parametrize("si", [0, 1, 2, 3, 6, 8])
def test_paired_stream_kernel_equals_unpaired(shape, si, monkeypatch):
    # HPAC_STREAM_PAIR=1: two logical threads per CUDA thread (opt-in variant)
    teams, tpt, ws, ipt, n = shape
    opts = E.make_bs_portfolio(n, 13)
    d_opts = dev(opts)
    grid = E.GridConfig(teams, tpt, ws, ipt)
    a = _run(grid, n, d_opts, SPECS[si])
    monkeypatch.setenv("HPAC_STREAM_PAIR", "1")
    b = _run(grid, n, d_opts, SPECS[si])
    for f in STAT_FIELDS:
        assert a[0].stats[f] == b[0].stats[f], f
    assert np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("si", [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12])
def test_lane_kernel_equals_tile_kernel(shape, si, monkeypatch):
    # bs_lane_kernel (default, barrier-free per-thread loads) vs bs_stream_kernel
    # (HPAC_STREAM_TMA=1, bulk-TMA staged team tiles): identical decisions,
    # stats, paths and outputs
    teams, tpt, ws, ipt, n = shape
    opts = E.make_bs_portfolio(n, 19)
    d_opts = dev(opts)
    grid = E.GridConfig(teams, tpt, ws, ipt)
    a = _run(grid, n, d_opts, SPECS[si])
    monkeypatch.setenv("HPAC_STREAM_TMA", "1")
    b = _run(grid, n, d_opts, SPECS[si])
    for f in STAT_FIELDS:
        assert a[0].stats[f] == b[0].stats[f], f
    assert np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])


@pytest.mark.parametrize("shape", [SHAPES[0], SHAPES[1], SHAPES[3], SHAPES[4]])
@pytest.mark.parametrize("spec_fn", [lambda: E.iact(1, 0.5), lambda: E.iact(2, 0.5),
                                     lambda: E.iact(4, 0.3, None, "warp"), lambda: E.iact(8, 0.2),
                                     lambda: E.iact(2, float("inf"), None, "warp"),
                                     lambda: E.iact(4, 0.0)])
def test_iact_lane_tables_equal_shared_tables(shape, spec_fn, monkeypatch):
    # per-lane tables in registers (bs_iact_lane_kernel) vs shared-memory
    # tables (bs_iact_kernel, HPAC_IACT_LANE=0) vs the lockstep engine
    teams, tpt, ws, ipt, n = shape
    opts = E.make_bs_portfolio(n, 17)
    d_opts = dev(opts)
    grid = E.GridConfig(teams, tpt, ws, ipt)
    try:
        a = _run(grid, n, d_opts, spec_fn)
    except E.ArenaOverflowError:
        # the reference's arena charge applies whatever the engine
        monkeypatch.setenv("HPAC_IACT_LANE", "0")
        with pytest.raises(E.ArenaOverflowError):
            _run(grid, n, d_opts, spec_fn)
        return
    monkeypatch.setenv("HPAC_IACT_LANE", "0")
    b = _run(grid, n, d_opts, spec_fn)
    c = _run(grid, n, d_opts, spec_fn, engine="thread")
    for r in (b, c):
        for f in STAT_FIELDS:
            assert a[0].stats[f] == r[0].stats[f], f
        assert np.array_equal(a[1], r[1])
        assert np.array_equal(a[2], r[2])


@pytest.mark.parametrize("spec_fn", [lambda: E.iact(2, 0.5), lambda: E.iact(4, 0.3, None, "warp"),
                                     lambda: E.iact(8, 0.2), lambda: E.iact(1, 0.5, None, "warp")])
@pytest.mark.parametrize("shape", [(8, 64, 32, 50, 8 * 64 * 50 - 37), (5, 32, 8, 97, 5 * 32 * 97)])
def test_iact_lane_tables_across_chunks(shape, spec_fn, monkeypatch):
    # more than 32 steps per thread: the lane-table kernel decides in chunks of
    # 32 and carries each slot's price across chunks (hits on older producers)
    teams, tpt, ws, ipt, n = shape
    opts = E.make_bs_portfolio(n, 23)
    d_opts = dev(opts)
    grid = E.GridConfig(teams, tpt, ws, ipt)
    a = _run(grid, n, d_opts, spec_fn)
    b = _run(grid, n, d_opts, spec_fn, engine="thread")
    for f in STAT_FIELDS:
        assert a[0].stats[f] == b[0].stats[f], f
    assert np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])
    if teams * tpt == 512:  # G = the portfolio's 512-option base block: hits every step
        assert a[0].stats["approx_invocations"] > 0


@pytest.mark.parametrize("level", ["thread", "warp"])
def test_iact_hit_threshold_edges(level, monkeypatch):
    """Hit iff sqrt_rn(ssq) <= thr: the iACT engines test ssq <= thr2 (the
    largest ssq whose rounded root is <= thr, found on the host) and take
    square roots only for near-ties. Pairs of options differing in the spot
    only, thresholds at the rounded distance and one ulp either side: every
    engine must match the lockstep engine's IEEE sqrt decisions."""
    rng = np.random.default_rng(3)
    tpt, ws, ipt = 32, 32, 2
    teams = 64
    n = teams * tpt * ipt
    G = teams * tpt
    base = E.make_bs_portfolio(G, 9)
    deltas = rng.uniform(1e-3, 1.0, G)
    second = base.copy()
    second[:, 0] += deltas  # step 1 record = step 0 record + delta in S
    opts = np.concatenate([base, second])
    d_opts = dev(opts)
    grid = E.GridConfig(teams, tpt, ws, ipt)
    dist = np.sqrt((second[:, 0] - base[:, 0]) ** 2)  # what the engines compute (5 dims, 4 zero)
    for thr in [float(np.median(dist)), float(np.nextafter(np.median(dist), 0)),
                float(np.nextafter(np.median(dist), 1))]:
        spec = lambda: E.iact(1, thr, None, level)
        a = _run(grid, n, d_opts, spec)
        monkeypatch.setenv("HPAC_IACT_LANE", "0")
        b = _run(grid, n, d_opts, spec)
        monkeypatch.delenv("HPAC_IACT_LANE")
        c = _run(grid, n, d_opts, spec, engine="thread")
        for r in (b, c):
            assert np.array_equal(a[2], r[2])
            assert np.array_equal(a[1], r[1])
        if level == "thread":
            want = (dist <= thr).astype(np.uint8)
            assert np.array_equal(a[2][G:], want)
