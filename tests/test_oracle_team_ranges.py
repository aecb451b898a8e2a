"""The checker's team-range runs (oracle_run_region_teams, the counterpart of
hpac_launch_t.team_begin/team_end) against its own whole-grid runs, which
test_oracle_vs_reference.py pins to the reference: splitting the logical
grid's teams into contiguous ranges, each keeping the global stride
(machine.hpp:77-84), must reproduce the whole run's outputs, paths and
summed stats exactly. This is the §8(e) decision-invariant split the
multi-GPU path uses, and what the full-shape GPU tests sample with."""
import numpy as np
import pytest

import oracle
from cases import random_case

SUMMED = ["total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps",
          "resident_warps"]


@pytest.mark.parametrize("seed", range(4))
def test_team_ranges_partition_the_whole_run(seed):
    rng = np.random.default_rng(7000 + seed)
    checked = 0
    for it in range(80):
        case = random_case(rng)
        w_out = case.init.copy()
        w_p = np.zeros(case.n, np.uint8)
        rc, st, msg = oracle.oracle_run(case.grid, case.n, case.mapping, case.region(w_out), case.spec, w_p)
        if rc != 0:
            continue
        T = case.grid.num_teams
        cuts = sorted(set([0, T] + list(rng.integers(0, T + 1, size=rng.integers(1, 4)))))
        r_out = case.init.copy()
        r_p = np.zeros(case.n, np.uint8)
        tot = {f: 0 for f in SUMMED}
        for b, e in zip(cuts[:-1], cuts[1:]):
            rc2, st2, msg2 = oracle.oracle_run_teams(case.grid, case.n, case.mapping, case.region(r_out),
                                                     case.spec, (b, e), r_p)
            assert rc2 == 0, (case.describe(), msg2)
            for f in SUMMED:
                tot[f] += getattr(st2, f)
        ctx = f"seed={seed} it={it} {case.describe()} cuts={cuts}"
        for f in SUMMED:
            assert tot[f] == getattr(st, f), (f, ctx)
        assert np.array_equal(r_out, w_out), ctx
        assert np.array_equal(r_p, w_p), ctx
        checked += 1
    assert checked >= 20


def test_team_range_outside_grid_is_config_error():
    case = random_case(np.random.default_rng(3))
    out = case.init.copy()
    rc, _, msg = oracle.oracle_run_teams(case.grid, case.n, case.mapping, case.region(out), case.spec,
                                         (0, case.grid.num_teams + 1))
    assert rc == 1 and "team range" in msg


def test_vectorised_prices_equal_scalar():
    from paper_2308_16877_b200 import engine as E
    opts = E.make_binomial_portfolio(64, 5)
    v = oracle.binomial_prices(opts, 96)
    import ctypes as C
    L = oracle.oracle()
    for i in range(0, 64, 7):
        x = C.c_double()
        assert L.oracle_binomial_price(opts[i].ctypes.data, 96, 1, 1, C.byref(x)) == 0
        assert x.value == v[i]
    bs = E.make_bs_portfolio(4096, 3)
    pv = oracle.bs_prices(bs)
    x = C.c_double()
    for i in range(0, 4096, 311):
        assert L.oracle_black_scholes_call(bs[i].ctypes.data, C.byref(x)) == 0
        assert x.value == pv[i]


@pytest.mark.ref
def test_threaded_reference_binomial_prices(ref_lib):
    from paper_2308_16877_b200 import engine as E
    opts = E.make_binomial_portfolio(48, 9)
    a = oracle.ref_binomial_prices(opts, 64, threads=4)
    b = oracle.binomial_prices(opts, 64)
    assert np.allclose(a, b, rtol=1e-12, atol=0)
