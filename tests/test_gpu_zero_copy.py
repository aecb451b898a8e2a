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
