"""The K-Means region's warp-cooperative FP64 tensor-op filter
(apps.cuh AppKmeans::warp_eval, EngineParams::warp_eval): labels, approx
counts and per-item paths must equal the CPU oracle (bench/kmeans.hpp:85-121
argmin; engine.hpp decisions) under every technique and decision level, on
ragged tails, several team sizes and k, and must equal the per-lane
CUDA-core filter (HPAC_KM_DMMA=0) bit for bit."""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2308_16877_b200 import engine as E
from gpu_util import dev

pytestmark = pytest.mark.gpu


def _blobs(n, d, k, seed, sep=6.0):
    rng = np.random.default_rng(seed)
    centres = rng.standard_normal((k, d)) * sep
    pts = centres[rng.integers(0, k, n)] + rng.standard_normal((n, d))
    return pts, pts[:k].copy()


def _run_gpu(pts, cents, grid, mp, spec, dmma=True):
    n = len(pts)
    lab = torch.full((n,), -7, dtype=torch.int32, device="cuda")
    paths = torch.zeros(n, dtype=torch.uint8, device="cuda")
    old = os.environ.get("HPAC_KM_DMMA")
    os.environ["HPAC_KM_DMMA"] = "1" if dmma else "0"
    try:
        r = E.run_region(grid, n, mp, E.kmeans_region(dev(pts), dev(cents), lab), spec, paths=paths)
    finally:
        if old is None:
            del os.environ["HPAC_KM_DMMA"]
        else:
            os.environ["HPAC_KM_DMMA"] = old
    return lab.cpu().numpy(), r.stats, paths.cpu().numpy()


def _run_oracle(pts, cents, grid, mp, spec):
    n = len(pts)
    lab = np.full(n, -7, np.int32)
    paths = np.zeros(n, np.uint8)
    rc, st, msg = oracle.oracle_run(grid, n, mp, E.kmeans_region(pts, cents, lab), spec, paths)
    assert rc == 0, msg
    return lab, st, paths


SPECS = {
    "exact": lambda: None,
    "small4": lambda: E.perfo("small", 4),
    "large2_warp": lambda: E.perfo("large", 2, level="warp"),
    "random40": lambda: E.perfo("random", 40, seed=11),
    "random50_warp": lambda: E.perfo("random", 50, level="warp", seed=3),
    "random52_team": lambda: E.perfo("random", 52, level="team", seed=5),
    "ini30": lambda: E.perfo("ini", 30),
    "iact": lambda: E.iact(2, 0.5, tables_per_warp=1),
    "iact_team": lambda: E.iact(4, 2.0, tables_per_warp=2, level="team"),
}


@pytest.mark.parametrize("spec", sorted(SPECS))
@pytest.mark.parametrize("shape", [(64 * 40 * 4, 64, 64), (5000 + 13, 64, 64), (3001, 32, 16),
                                   (4099, 96, 8), (2048 + 5, 128, 72)])
def test_dmma_filter_matches_oracle(spec, shape):
    n, tpt, k = shape
    pts, cents = _blobs(n, 32, k, seed=n + k)
    grid, mp = E.resolve_grid("kmeans", n, threads_per_team=tpt, items_per_thread=4)
    sp = SPECS[spec]()
    got, gst, gpaths = _run_gpu(pts, cents, grid, mp, sp)
    want, ost, opaths = _run_oracle(pts, cents, grid, mp, sp)
    assert np.array_equal(got, want), int(np.sum(got != want))
    assert gst["approx_invocations"] == ost.approx_invocations
    assert gst["total_invocations"] == ost.total_invocations
    assert gst["divergent_warp_steps"] == ost.divergent_warp_steps
    assert np.array_equal(gpaths, opaths)


@pytest.mark.parametrize("case", ["duplicates", "equidistant", "nonfinite", "huge"])
def test_dmma_equals_cuda_core_filter(case):
    rng = np.random.default_rng(17)
    n, d, k = 64 * 32 * 4 + 9, 32, 64
    cents = rng.standard_normal((k, d)) * 3.0
    pts = rng.standard_normal((n, d)) * 3.0
    if case == "duplicates":
        cents[5] = cents[9]
        pts[: n // 2] = cents[rng.integers(0, k, n // 2)]
    elif case == "equidistant":
        a, b = rng.integers(0, k, n), rng.integers(0, k, n)
        pts = 0.5 * (cents[a] + cents[b])
    elif case == "nonfinite":
        pts[::97, 3] = np.nan
        pts[::89, 7] = np.inf
        cents[17, 0] = np.nan
    elif case == "huge":
        pts, cents = pts * 1e150, cents * 1e150
    grid, mp = E.resolve_grid("kmeans", n, items_per_thread=4)
    a, _, _ = _run_gpu(pts, cents, grid, mp, None, dmma=True)
    b, _, _ = _run_gpu(pts, cents, grid, mp, None, dmma=False)
    want, _, _ = _run_oracle(pts, cents, grid, mp, None)
    assert np.array_equal(a, b), int(np.sum(a != b))
    assert np.array_equal(a, want)


@pytest.mark.parametrize("n", [1, 5, 31, 33, 64 * 4 + 1])
def test_dmma_tiny_and_ragged_n(n):
    pts, _ = _blobs(max(n, 64), 32, 64, seed=n)
    pts = pts[:n].copy()
    cents = _blobs(64, 32, 64, seed=99)[1]
    grid, mp = E.resolve_grid("kmeans", n, items_per_thread=4)
    got, gst, gpaths = _run_gpu(pts, cents, grid, mp, None)
    want, ost, opaths = _run_oracle(pts, cents, grid, mp, None)
    assert np.array_equal(got, want)
    assert gst["total_invocations"] == ost.total_invocations == n
