"""The binomial decide -> price -> resolve launch (csrc/engine_team.cu,
launch_bino_pipeline) and the 8-teams-per-CTA TAF kernel against the
one-kernel chunked engine (HPAC_BINO_PIPELINE=0) and the oracle: identical stats, path bits and prices
for exact, iACT and perforation runs, American/European puts and calls,
lattices below and above the register bound, ragged grids and team ranges.
Both engines price an option with the same function of the option alone
(binomial_put_seg / binomial_warp_price), so the prices must be bit-equal."""
import numpy as np
import pytest
import torch

import oracle
from paper_2308_16877_b200 import engine as E
from gpu_util import dev

pytestmark = pytest.mark.gpu

STAT_FIELDS = ["total_invocations", "approx_invocations", "divergent_warp_steps",
               "total_warp_steps", "resident_warps"]


def _run(grid, n, d_opts, steps, spec_fn, pipeline, monkeypatch, am=True, put=True, team_range=None):
    monkeypatch.setenv("HPAC_BINO_PIPELINE", "1" if pipeline else "0")
    out = torch.full((n,), -7.0, dtype=torch.float64, device="cuda")
    paths = torch.zeros(n, dtype=torch.uint8, device="cuda")
    lr = E.run_region(grid, n, 1, E.binomial_region(d_opts, steps, out, american=am, put=put),
                      spec_fn(), paths=paths, team_range=team_range)
    return lr, out.cpu().numpy(), paths.cpu().numpy()


CASES = [  # (teams, ipt, n, lattice steps)
    (40, 24, 40 * 24, 64),
    (13, 37, 13 * 37 - 5, 256),
    (64, 16, 64 * 16, 1024),
    (7, 9, 7 * 9, 1100),
]
SPECS = [lambda: None, lambda: E.iact(4, 0.4, level="team"), lambda: E.iact(1, 0.0, level="team"),
         lambda: E.iact(8, float("inf"), level="team"), lambda: E.perfo("small", 3),
         lambda: E.perfo("random", 40, seed=3),
         # TAF: 8 teams per CTA (binomial_taf_seg_kernel) vs one team per CTA
         lambda: E.taf(2, 4, 0.01, "team"), lambda: E.taf(3, 2, float("inf"), "team"),
         lambda: E.taf(5, 1, 0.5, "team")]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("si", range(len(SPECS)))
def test_pipeline_equals_chunked_engine(case, si, monkeypatch):
    teams, ipt, n, steps = case
    opts = E.make_binomial_portfolio(n, 19)
    d = dev(opts)
    grid = E.GridConfig(teams, 64, 32, ipt)
    a = _run(grid, n, d, steps, SPECS[si], True, monkeypatch)
    b = _run(grid, n, d, steps, SPECS[si], False, monkeypatch)
    for f in STAT_FIELDS:
        assert a[0].stats[f] == b[0].stats[f], f
    assert np.array_equal(a[2], b[2])
    assert np.array_equal(a[1], b[1])


@pytest.mark.parametrize("am,put", [(True, False), (False, True), (False, False)])
def test_pipeline_other_payoffs(am, put, monkeypatch):
    n, steps = 20 * 16, 200
    opts = E.make_binomial_portfolio(n, 23)
    d = dev(opts)
    grid = E.GridConfig(20, 64, 32, 16)
    for spec_fn in (lambda: None, lambda: E.iact(4, 0.4, level="team")):
        a = _run(grid, n, d, steps, spec_fn, True, monkeypatch, am, put)
        b = _run(grid, n, d, steps, spec_fn, False, monkeypatch, am, put)
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_pipeline_team_ranges_compose(monkeypatch):
    # two team ranges of one logical grid == the whole launch (§8e split)
    n, steps = 50 * 20, 128
    opts = E.make_binomial_portfolio(n, 29)
    d = dev(opts)
    grid = E.GridConfig(50, 64, 32, 20)
    spec = lambda: E.iact(4, 0.4, level="team")
    whole = _run(grid, n, d, steps, spec, True, monkeypatch)
    monkeypatch.setenv("HPAC_BINO_PIPELINE", "1")
    out = torch.full((n,), -7.0, dtype=torch.float64, device="cuda")
    tot = {f: 0 for f in STAT_FIELDS}
    for tr in [(0, 21), (21, 50)]:
        lr = E.run_region(grid, n, 1, E.binomial_region(d, steps, out), spec(), team_range=tr)
        for f in STAT_FIELDS:
            tot[f] += lr.stats[f]
    assert np.array_equal(out.cpu().numpy(), whole[1])
    for f in STAT_FIELDS:
        assert tot[f] == whole[0].stats[f], f


def test_pipeline_vs_oracle_replay(monkeypatch):
    n, steps = 30 * 40, 512
    opts = E.make_binomial_portfolio(n, 31)
    d = dev(opts)
    grid = E.GridConfig(30, 64, 32, 40)
    ex = _run(grid, n, d, steps, lambda: None, True, monkeypatch)[1]
    lr, g_out, g_paths = _run(grid, n, d, steps, lambda: E.iact(4, 0.4, level="team"), True, monkeypatch)
    o_out = np.zeros(n)
    o_paths = np.zeros(n, np.uint8)
    rc, st, msg = oracle.oracle_run(grid, n, 1, E.table_region(opts, ex.reshape(n, 1), o_out),
                                    E.iact(4, 0.4, level="team"), o_paths)
    assert rc == 0, msg
    for f in STAT_FIELDS:
        assert lr.stats[f] == getattr(st, f), f
    assert np.array_equal(g_paths, o_paths)
    assert np.array_equal(g_out, o_out)


@pytest.mark.parametrize("steps", [256, 1024])
def test_segmented_lattice_wide_parameter_range(steps, monkeypatch):
    """American puts far from the C2 portfolio (vol 0.05-1.2, T 0.05-5,
    r -0.01-0.08, moneyness 0.3-3; all valid CRR lattices): the 8-lane segmented lattice and its
    whole-warp fallbacks stay within 1e-6 of the CPU lattice, and the exact
    and iACT runs price every option identically."""
    rng = np.random.default_rng(5)
    n = 640
    S = rng.uniform(20, 200, n)
    opts = np.stack([S, S * np.exp(rng.uniform(np.log(0.3), np.log(3.0), n)), rng.uniform(-0.01, 0.08, n),
                     rng.uniform(0.05, 1.2, n), rng.uniform(0.05, 5.0, n)], axis=1)
    d = dev(opts)
    grid = E.GridConfig(40, 64, 32, 16)
    lr, out, _ = _run(grid, n, d, steps, lambda: None, True, monkeypatch)
    want = oracle.binomial_prices(opts, steps)
    rel = np.abs(out - want) / np.maximum(np.abs(want), 1e-300)
    ok = (rel <= 1e-6) | (np.abs(out - want) <= 1e-12 * opts[:, 1])
    assert ok.all(), (rel.max(), np.argmax(rel))
    _, o2, p2 = _run(grid, n, d, steps, lambda: E.iact(2, 0.0, level="team"), True, monkeypatch)
    assert np.array_equal(o2[p2 == 0], out[p2 == 0])
