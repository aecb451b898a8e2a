"""TAF decisions at the threshold edge. The device RSD test first decides
with a division-free estimate and falls back to the exact two-pass RSD
(taf.hpp:29-40) near the threshold (hpac_device.cuh taf_window_passes);
these windows sit exactly on, one ulp around, and within 1e-13 of the
threshold, so any disagreement between the estimate's margin and the
exact test shows up as a decision mismatch against the oracle."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from paper_2308_16877_b200 import engine as E

pytestmark = pytest.mark.gpu

STAT_FIELDS = ["total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps"]


def _rsd(w):
    L = oracle.oracle()
    a = np.ascontiguousarray(w, dtype=np.float64)
    return L.oracle_rsd(a.ctypes.data, len(a))


@pytest.mark.parametrize("h", [2, 3, 5])
@pytest.mark.parametrize("out_dims", [1, 2])
def test_taf_threshold_edge_bit_exact(h, out_dims):
    rng = np.random.default_rng(h * 10 + out_dims)
    teams, tpt, steps = 8, 64, h + 2
    T = teams * tpt
    n = T * steps
    base = 1.0 + 0.3 * rng.standard_normal(h)
    thr = _rsd(base)
    # per-thread first windows: exact power-of-two copies of `base` (same
    # rsd), sign flips, one-ulp perturbations, and 1e-13 relative jitters
    vals = np.empty((steps, T, out_dims))
    for t in range(T):
        kind = t % 4
        w = base * 2.0 ** ((t // 4) % 40 - 20)
        if kind == 1:
            w = -w
        elif kind == 2:
            w = w.copy()
            w[t % h] = np.nextafter(w[t % h], np.inf if (t // 8) % 2 else -np.inf)
        elif kind == 3:
            w = w * (1.0 + 1e-13 * rng.standard_normal(h))
        for d in range(out_dims):
            vals[:h, t, d] = w if d == 0 else w[::-1] * (1 + d)
        vals[h:, t, :] = rng.standard_normal((steps - h, out_dims))
    table = vals.reshape(n, out_dims)  # item = t + step*T (grid-stride order)
    for sign in (0.0, -1.0, 1.0):
        th = thr if sign == 0 else np.nextafter(thr, sign * np.inf)
        spec = lambda: E.taf(h, 2, th)
        grid = E.GridConfig(teams, tpt, 32, steps)
        out = torch.zeros((n, out_dims), dtype=torch.float64, device="cuda")
        paths = torch.zeros(n, dtype=torch.uint8, device="cuda")
        reg = E.table_region(None, torch.from_numpy(table).cuda(), out, input_dims=0, output_dims=out_dims)
        lr = E.run_region(grid, n, 0, reg, spec(), paths=paths)
        o_out = np.zeros((n, out_dims))
        o_paths = np.zeros(n, np.uint8)
        rc, st, msg = oracle.oracle_run(grid, n, 0, E.table_region(None, table, o_out, input_dims=0,
                                                                   output_dims=out_dims), spec(), o_paths)
        assert rc == 0, msg
        for f in STAT_FIELDS:
            assert lr.stats[f] == getattr(st, f), (f, sign)
        assert np.array_equal(paths.cpu().numpy(), o_paths), sign
        assert np.array_equal(out.cpu().numpy(), o_out), sign
        # the edge is really exercised: some threads pass, some fail
        first_pred = o_paths.reshape(steps, T)[h]
        if out_dims == 1 and sign == 0:
            assert 0 < first_pred.sum() < T
