"""The K-Means region's filtered argmin (apps.cuh AppKmeans::eval): labels
from the |x|^2 + |c|^2 - 2 x.c estimate must equal the reference's argmin of
sqrt(no-FMA dimension-order sums) with strict < / lowest index
(bench/kmeans.hpp:85-121) — including the cases the filter hands to the exact
path: duplicate centroids (exact ties), points equidistant from two
centroids, near-ties below the error bound, and non-finite data."""
import numpy as np
import pytest
import torch

import oracle
from paper_2308_16877_b200 import engine as E
from gpu_util import dev

pytestmark = pytest.mark.gpu


def _labels_gpu(pts, cents, ipt=4):
    n = len(pts)
    lab = torch.full((n,), -7, dtype=torch.int32, device="cuda")
    grid, mp = E.resolve_grid("kmeans", n, items_per_thread=ipt)
    E.run_region(grid, n, mp, E.kmeans_region(dev(pts), dev(cents), lab), None)
    return lab.cpu().numpy(), grid


def _labels_oracle(pts, cents, grid):
    n = len(pts)
    lab = np.full(n, -7, np.int32)
    rc, st, msg = oracle.oracle_run(grid, n, 0, E.kmeans_region(pts, cents, lab), None)
    assert rc == 0, msg
    return lab


@pytest.mark.parametrize("case", ["random", "duplicates", "equidistant", "near_tie", "nonfinite", "huge"])
def test_filtered_argmin_matches_reference(case):
    rng = np.random.default_rng(7)
    n, d, k = 64 * 64 * 4, 32, 64
    cents = rng.standard_normal((k, d)) * 3.0
    pts = rng.standard_normal((n, d)) * 3.0
    if case == "duplicates":
        cents[5] = cents[9]
        cents[40] = cents[2]
        pts[: n // 2] = cents[rng.integers(0, k, n // 2)] + 1e-9 * rng.standard_normal((n // 2, d))
    elif case == "equidistant":
        # midpoints of centroid pairs: exact or ulp-level ties
        a, b = rng.integers(0, k, n), rng.integers(0, k, n)
        pts = 0.5 * (cents[a] + cents[b])
    elif case == "near_tie":
        a, b = rng.integers(0, k, n), rng.integers(0, k, n)
        t = 0.5 + rng.standard_normal(n)[:, None] * 1e-13
        pts = cents[a] * t + cents[b] * (1 - t)
    elif case == "nonfinite":
        pts[::97, 3] = np.nan
        pts[::89, 7] = np.inf
        cents[17, 0] = np.nan
    elif case == "huge":
        pts = pts * 1e150
        cents = cents * 1e150
    got, grid = _labels_gpu(pts, cents)
    want = _labels_oracle(pts, cents, grid)
    assert np.array_equal(got, want), int(np.sum(got != want))


def test_filtered_argmin_nan_first_centroid_keeps_label_zero():
    """A NaN distance to centroid 0 makes every later strict < fail in the
    reference (best stays 0)."""
    rng = np.random.default_rng(3)
    n, d, k = 64 * 16 * 4, 32, 64
    cents = rng.standard_normal((k, d))
    cents[0, 0] = np.nan
    pts = rng.standard_normal((n, d))
    got, grid = _labels_gpu(pts, cents)
    want = _labels_oracle(pts, cents, grid)
    assert np.array_equal(got, want)
    assert np.all(want == 0)
