"""Two VERDICT r01 items on the device:

* the quality metrics hpac_mape / hpac_mcr against the reference's own
  mape / mcr (metrics.hpp:17-45) on identical arrays, including the zero
  policy (0/0 -> 0; accurate 0 with approximate != 0 -> infinity);
* the §8(e) decision-invariant multi-GPU split: N launches over contiguous
  team ranges of ONE logical grid (hpac_launch_t.team_begin/team_end, the
  global stride kept, machine.hpp:77-84) reproduce the whole-grid run bit
  for bit, at the headline shape. This is what bench.py runs per rank at N>1.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2308_16877_b200 import engine as E
from gpu_util import dev

pytestmark = pytest.mark.gpu

SUMMED = ["total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps",
          "resident_warps", "lattice_nodes", "lattice_fallbacks"]


def _ref_mape(a, b):
    if oracle.ref_available():
        return oracle.ref().ref_mape(a.ctypes.data, b.ctypes.data, len(a))
    return oracle.oracle().oracle_mape(a.ctypes.data, b.ctypes.data, len(a))


def _ref_mcr(a, b):
    if oracle.ref_available():
        return oracle.ref().ref_mcr(a.ctypes.data, b.ctypes.data, len(a))
    return oracle.oracle().oracle_mcr(a.ctypes.data, b.ctypes.data, len(a))


@pytest.mark.parametrize("n", [1, 7, 1000, 1 << 20, (1 << 22) + 13])
def test_mape_matches_reference(n):
    rng = np.random.default_rng(n)
    a = rng.uniform(-50, 50, n)
    b = a * (1 + rng.normal(0, 0.01, n))
    b[::5] = a[::5]
    if n > 10:
        a[3] = 0.0
        b[3] = 0.0  # 0/0 contributes 0
    got = E.mape(dev(a), dev(b))
    want = _ref_mape(a, b)
    assert abs(got - want) <= 1e-12 * abs(want) + 1e-300, (got, want)


def test_mape_zero_policy():
    a = np.array([0.0, 1.0, 2.0, 0.0])
    b = np.array([0.0, 1.0, 2.5, 0.0])
    assert E.mape(dev(a), dev(b)) == _ref_mape(a, b) == 0.5 / 2.0 / 4
    b2 = b.copy()
    b2[0] = 1e-300  # accurate 0, approximate != 0 -> infinity
    assert _ref_mape(a, b2) == np.inf
    assert E.mape(dev(a), dev(b2)) == np.inf
    e = np.zeros(0)
    assert E.mape(torch.zeros(0, dtype=torch.float64, device="cuda"),
                  torch.zeros(0, dtype=torch.float64, device="cuda")) == _ref_mape(e, e) == 0.0


@pytest.mark.parametrize("n", [1, 1000, (1 << 24) + 5])
def test_mcr_matches_reference(n):
    rng = np.random.default_rng(n + 1)
    a = rng.integers(0, 64, n).astype(np.int32)
    b = a.copy()
    flip = rng.random(n) < 0.013
    b[flip] = (b[flip] + 1) % 64
    assert E.mcr(dev(a), dev(b)) == _ref_mcr(a, b)


def _split_equals_whole(grid, n, mapping, region_fn, spec, out_like, parts):
    whole = torch.zeros_like(out_like)
    wp = torch.zeros(n, dtype=torch.uint8, device="cuda")
    lw = E.run_region(grid, n, mapping, region_fn(whole), spec, paths=wp)
    T = grid.num_teams
    split = torch.zeros_like(out_like)
    sp_ = torch.zeros(n, dtype=torch.uint8, device="cuda")
    tot = {f: 0 for f in SUMMED}
    for r in range(parts):
        lr = E.run_region(grid, n, mapping, region_fn(split), spec, paths=sp_,
                          team_range=(r * T // parts, (r + 1) * T // parts))
        for f in SUMMED:
            tot[f] += lr.stats[f]
    for f in SUMMED:
        assert tot[f] == lw.stats[f], (f, tot[f], lw.stats[f])
    assert torch.equal(split, whole)
    assert torch.equal(sp_, wp)
    return lw


@pytest.mark.parametrize("parts", [2, 8])
def test_headline_team_range_split(parts):
    """C2 at its full shape as N 'GPUs' (team ranges) vs one: identical."""
    n = 1 << 20
    opts = dev(E.make_binomial_portfolio(n, 42))
    grid, mapping = E.resolve_grid("binomial", n, items_per_thread=384)
    lw = _split_equals_whole(grid, n, mapping, lambda o: E.binomial_region(opts, 1024, o),
                             E.iact(4, 0.4, level="team"), torch.zeros(n, dtype=torch.float64, device="cuda"),
                             parts)
    assert lw.stats["approx_invocations"] > 0


@pytest.mark.parametrize("spec_fn", [lambda: None, lambda: E.taf(5, 1, 0.5), lambda: E.taf(5, 8, 0.5, "team"),
                                     lambda: E.iact(2, 0.5)])
def test_blackscholes_team_range_split(spec_fn):
    n = 1 << 22
    opts = dev(E.make_bs_portfolio(n, 42))
    grid, mapping = E.resolve_grid("blackscholes", n)
    _split_equals_whole(grid, n, mapping, lambda o: E.blackscholes_region(opts, o), spec_fn(),
                        torch.zeros(n, dtype=torch.float64, device="cuda"), 8)


def test_kmeans_region_team_range_split():
    n, d, k = 1 << 20, 32, 64
    pts = E.make_blobs(n, d, k, 42, 30.0)
    dp, dc = dev(pts), dev(pts[:k])
    grid, mapping = E.resolve_grid("kmeans", n)
    _split_equals_whole(grid, n, mapping, lambda o: E.kmeans_region(dp, dc, o),
                        E.perfo("random", 52, level="team"), torch.zeros(n, dtype=torch.int32, device="cuda"), 4)
