"""CUDA engine vs the C restatement on randomised pure regions.

Bit-exact bar (integer/index work and decisions on replayed values):
status, arena/barrier error details, total/approx invocations, divergent and
total warp steps, resident warps, per-item path bits and every output value.
"""
import numpy as np
import pytest

import oracle
from cases import random_case

pytestmark = pytest.mark.gpu

STAT_FIELDS = ["total_invocations", "approx_invocations", "divergent_warp_steps",
               "total_warp_steps", "resident_warps"]


def _check(case, ctx):
    from gpu_util import run_case_gpu
    g_status, g_stats, g_out, g_paths, g_msg = run_case_gpu(case)
    o_out = case.init.copy()
    o_paths = np.zeros(case.n, np.uint8)
    o_rc, o_st, o_msg = oracle.oracle_run(case.grid, case.n, case.mapping, case.region(o_out),
                                          case.spec, o_paths)
    ctx = f"{ctx} {case.describe()} gpu={g_msg!r} oracle={o_msg!r}"
    assert g_status == o_rc, ctx
    if o_rc == 2:
        assert g_stats["arena_required"] == o_st.arena_required, ctx
        assert g_stats["arena_available"] == o_st.arena_available, ctx
    elif o_rc == 3:
        assert (g_stats["fail_team"], g_stats["fail_step"], g_stats["fail_missing"]) == \
            (o_st.fail_team, o_st.fail_step, o_st.fail_missing), ctx
    elif o_rc == 0:
        for f in STAT_FIELDS:
            assert g_stats[f] == getattr(o_st, f), (f, ctx)
        assert np.array_equal(g_out, o_out), ctx
        assert np.array_equal(g_paths, o_paths), ctx


@pytest.mark.parametrize("seed", range(8))
def test_random_regions_bit_exact(seed):
    rng = np.random.default_rng(77 + seed)
    for it in range(60):
        case = random_case(rng, allow_random_perfo=True)
        _check(case, f"seed={seed} it={it}")


@pytest.mark.parametrize("seed", range(3))
def test_random_regions_wide_teams(seed):
    """Bigger teams (up to 1024 threads) and more teams."""
    rng = np.random.default_rng(900 + seed)
    for it in range(15):
        case = random_case(rng, allow_random_perfo=True, max_threads=1024)
        _check(case, f"wide seed={seed} it={it}")
