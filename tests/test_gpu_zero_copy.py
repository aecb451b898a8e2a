"""hpac_run_region_host zero-copy (pinned caller buffers read/written in
place by the kernel) vs the staged path (HPAC_HOST_COPY=1) and vs the device
entry: identical outputs, labels and stats."""
import os

import numpy as np
import pytest
import torch

from paper_2308_16877_b200 import engine as E

pytestmark = pytest.mark.gpu


def _host_run(grid, n, mp, region, spec, staged):
    old = os.environ.get("HPAC_HOST_COPY")
    os.environ["HPAC_HOST_COPY"] = "1" if staged else "0"
    try:
        return E.run_region_host(grid, n, mp, region, spec)
    finally:
        if old is None:
            del os.environ["HPAC_HOST_COPY"]
        else:
            os.environ["HPAC_HOST_COPY"] = old


@pytest.mark.parametrize("spec_fn", [lambda: None, lambda: E.taf(5, 1, 0.5), lambda: E.taf(3, 4, 0.3, level="warp"),
                                     lambda: E.iact(2, 0.3), lambda: E.perfo("small", 4)])
@pytest.mark.parametrize("n", [64 * 16 * 20 + 7, 1 << 16])
def test_blackscholes_zero_copy(spec_fn, n):
    opts = E.make_bs_portfolio(n, 5)
    grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
    h_in = torch.from_numpy(opts).pin_memory()
    outs = []
    for staged in (False, True):
        h_out = torch.full((n,), -1.0, dtype=torch.float64).pin_memory()
        r = _host_run(grid, n, mp, E.blackscholes_region(h_in.numpy(), h_out.numpy()), spec_fn(), staged)
        assert r.stats["zero_copy"] == (0 if staged else 1)
        outs.append((h_out.clone(), r.stats))
    d_out = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
    rd = E.run_region(grid, n, mp, E.blackscholes_region(h_in.cuda(), d_out), spec_fn())
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][0], d_out.cpu())
    for key in ("total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps"):
        assert outs[0][1][key] == outs[1][1][key] == rd.stats[key], key


def test_pageable_buffers_stay_staged():
    n = 4096
    opts = E.make_bs_portfolio(n, 5)
    grid, mp = E.resolve_grid("blackscholes", n, items_per_thread=16)
    out = np.zeros(n)
    r = E.run_region_host(grid, n, mp, E.blackscholes_region(opts, out), None)
    assert r.stats["zero_copy"] == 0
    d_out = torch.zeros(n, dtype=torch.float64, device="cuda")
    E.run_region(grid, n, mp, E.blackscholes_region(torch.from_numpy(opts).cuda(), d_out), None)
    assert np.array_equal(out, d_out.cpu().numpy())


@pytest.mark.parametrize("spec_fn", [lambda: None, lambda: E.perfo("random", 50, level="warp", seed=2)])
def test_kmeans_labels_zero_copy(spec_fn):
    n, d, k = 64 * 4 * 64 + 11, 32, 64
    pts = E.make_blobs(n, d, k, 7, 8.0)
    grid, mp = E.resolve_grid("kmeans", n, items_per_thread=4)
    h_pts = torch.from_numpy(pts).pin_memory()
    cents = pts[:k].copy()
    labs = []
    for staged in (False, True):
        h_lab = torch.zeros(n, dtype=torch.int32).pin_memory()
        r = _host_run(grid, n, mp, E.kmeans_region(h_pts.numpy(), cents, h_lab.numpy()), spec_fn(), staged)
        assert r.stats["zero_copy"] == (0 if staged else 1)
        labs.append(h_lab.clone())
    assert torch.equal(labs[0], labs[1])


@pytest.mark.parametrize("spec_fn,keeps", [(lambda: None, False), (lambda: E.iact(4, 0.4, level="team"), False),
                                           (lambda: E.perfo("small", 3), True)])
def test_binomial_host_entry_outputs(spec_fn, keeps):
    # staged host entry: without perforation every item is written, so the
    # caller's output buffer is not copied in; perforation keeps skipped items
    n, steps = 24 * 16, 128
    opts = E.make_binomial_portfolio(n, 8)
    grid, mp = E.resolve_grid("binomial", n, items_per_thread=16)
    out = np.full(n, -7.0)
    r = E.run_region_host(grid, n, mp, E.binomial_region(opts, steps, out), spec_fn())
    d_out = torch.full((n,), -7.0, dtype=torch.float64, device="cuda")
    rd = E.run_region(grid, n, mp, E.binomial_region(torch.from_numpy(opts).cuda(), steps, d_out), spec_fn())
    assert np.array_equal(out, d_out.cpu().numpy())
    assert r.stats["approx_invocations"] == rd.stats["approx_invocations"]
    assert bool((out == -7.0).any()) == keeps


STATS = ["total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps",
         "resident_warps", "lattice_nodes"]


@pytest.mark.parametrize("app", ["binomial", "blackscholes"])
@pytest.mark.parametrize("spec_fn", [lambda: None, lambda: E.iact(4, 0.4, level="team"),
                                     lambda: E.taf(3, 2, 0.3, level="team"), lambda: E.perfo("small", 3)])
@pytest.mark.parametrize("pinned", [False, True])
def test_host_entry_team_ranges(app, spec_fn, pinned):
    # hpac_run_region_host_teams: the team ranges of one global grid, each
    # moving only its column block of items, compose to one device launch
    # (prices, paths of untouched items, summed stats); items outside a
    # range are neither read nor written
    if app == "binomial":
        grid, mp = E.resolve_grid("binomial", 41 * 20, items_per_thread=20)
        n = grid.num_teams * 20 - 17
        opts = E.make_binomial_portfolio(n, 21)
        mk = lambda i, o: E.binomial_region(i, 64, o)
    else:
        grid, mp = E.resolve_grid("blackscholes", 37 * 64 * 5, items_per_thread=5)
        n = grid.num_teams * grid.threads_per_team * 5 - 29
        opts = E.make_bs_portfolio(n, 21)
        mk = lambda i, o: E.blackscholes_region(i, o)
    d_out = torch.full((n,), -7.0, dtype=torch.float64, device="cuda")
    rd = E.run_region(grid, n, mp, mk(torch.from_numpy(opts).cuda(), d_out), spec_fn())
    h_in = torch.from_numpy(opts)
    h_out = torch.full((n,), -7.0, dtype=torch.float64)
    if pinned:
        h_in, h_out = h_in.pin_memory(), h_out.pin_memory()
    T = grid.num_teams
    cuts = [0, T // 3, T // 3 + 1, (2 * T) // 3, T]
    tot = {f: 0 for f in STATS}
    for a, b in zip(cuts[:-1], cuts[1:]):
        r = E.run_region_host(grid, n, mp, mk(h_in.numpy(), h_out.numpy()), spec_fn(), team_range=(a, b))
        for f in STATS:
            tot[f] += r.stats[f]
        if a == 0:  # after the first range only its items changed
            got = h_out.numpy().copy()
            w = 1 if app == "binomial" else grid.threads_per_team
            G = T * w
            col = np.arange(n) % G
            inside = (col >= a * w) & (col < b * w)
            assert np.array_equal(got[inside], d_out.cpu().numpy()[inside])
            assert np.all(got[~inside] == -7.0)
    assert np.array_equal(h_out.numpy(), d_out.cpu().numpy())
    for f in STATS:
        assert tot[f] == rd.stats[f], f


def test_host_entry_team_range_rejects_other_regions():
    n, d, k = 64 * 4 * 4, 32, 8
    pts = E.make_blobs(n, d, k, 7, 8.0)
    grid, mp = E.resolve_grid("kmeans", n, items_per_thread=4)
    with pytest.raises(E.UnsupportedError):
        E.run_region_host(grid, n, mp, E.kmeans_region(pts, pts[:k].copy(), np.zeros(n, np.int32)),
                          None, team_range=(0, 1))
