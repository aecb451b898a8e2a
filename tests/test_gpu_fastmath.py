"""csrc/fastmath.cuh on the device (hpac_fm_eval): the ulp bounds of
test_fastmath.py against mpmath, and Blackscholes prices from the fastmath
formula against the libdevice formula (the round-1 kernel) on the C1
portfolio."""
import numpy as np
import pytest
import torch

from fastmath_ref import BOUNDS, reference, samples, ulp_errors
from paper_2308_16877_b200 import abi
from paper_2308_16877_b200 import engine as E

pytestmark = pytest.mark.gpu
KIND = {"exp": 0, "log": 1, "erfc": 2, "bs": 3, "ld_exp": 4, "ld_log": 5, "ld_erfc": 6, "ld_bs": 7}


def fm_eval(kind, x, n=None):
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    n = xd.numel() if n is None else n
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    rc = abi.lib().hpac_fm_eval(KIND[kind], xd.data_ptr(), y.data_ptr(), n, None)
    assert rc == 0
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("kind", ["exp", "log", "erfc"])
def test_device_ulp_bound(kind):
    x = samples(kind, seed=17)
    err = ulp_errors(fm_eval(kind, x), reference(kind, x))
    assert err.max() <= BOUNDS[kind], (kind, err.max(), x[err.argmax()])


def test_device_special_values():
    nan, inf = np.nan, np.inf
    y = fm_eval("erfc", [nan, -inf, inf, 30.0, -30.0, 0.0, 27.3])
    assert np.isnan(y[0]) and list(y[1:]) == [2.0, 0.0, 0.0, 2.0, 1.0, 0.0]
    y = fm_eval("log", [0.0, -1.0, inf, 1.0, 5e-320])
    assert y[0] == -inf and np.isnan(y[1]) and y[2] == inf and y[3] == 0.0
    assert abs(y[4] - np.log(5e-320)) <= np.spacing(abs(np.log(5e-320)))


def test_device_erfc_close_to_libdevice_dense():
    x = np.linspace(-6.0, 26.0, 1 << 20)
    a, b = fm_eval("erfc", x), fm_eval("ld_erfc", x)
    ulp = np.spacing(np.abs(b))
    assert np.all(np.abs(a - b) <= 8 * np.maximum(ulp, 5e-324))


def test_bs_prices_match_libdevice_formula():
    n = 1 << 20
    opts = E.make_bs_portfolio(n, 42)
    a, b = fm_eval("bs", opts, n), fm_eval("ld_bs", opts, n)
    spot = opts.reshape(n, 5)[:, 0]
    assert np.all(np.isfinite(a))
    assert np.all(np.abs(a - b) <= 1e-13 * spot + 1e-12 * np.abs(b)), np.max(np.abs(a - b))


def test_bs_fast_domain_edges_match_libdevice_formula():
    # apps.cuh bs_call prices inside an integer-tested box (spot, strike in
    # [2^-500, 2^500), vol < 2^8, maturity < 2^5, |rate| < 2^3) without the
    # per-step argument checks and falls back to bs_call_general outside it:
    # options on both sides of every edge, plus log-uniform random ones, agree
    # with the libdevice formula
    one_minus = 1.0 - 2.0 ** -52
    base = np.array([100.0, 95.0, 0.03, 0.2, 1.0])
    edges = {0: [2.0 ** -500, 2.0 ** -500 * one_minus, 2.0 ** 500 * one_minus, 2.0 ** 500, 1e-160, 1e160],
             1: [2.0 ** -500, 2.0 ** -500 * one_minus, 2.0 ** 500 * one_minus, 2.0 ** 500, 1e-160, 1e160],
             2: [-8.0 * one_minus, 8.0 * one_minus, 8.0, -8.0, 20.0, -0.5],
             3: [2.0 ** -500, 2.0 ** -500 * one_minus, 256.0 * one_minus, 256.0, 300.0, 1e-200],
             4: [2.0 ** -500, 2.0 ** -500 * one_minus, 32.0 * one_minus, 32.0, 40.0, 1e-200]}
    rows = []
    for col, vals in edges.items():
        for v in vals:
            r = base.copy()
            r[col] = v
            if col == 0:
                r[1] = v * 0.95
            rows.append(r)
    rng = np.random.default_rng(5)
    m = 1 << 16
    rnd = np.stack([10.0 ** rng.uniform(-3, 3, m), 10.0 ** rng.uniform(-3, 3, m),
                    rng.uniform(-20, 20, m), 10.0 ** rng.uniform(-4, 2.6, m),
                    10.0 ** rng.uniform(-4, 1.7, m)], axis=1)
    opts = np.concatenate([np.array(rows), rnd])
    n = len(opts)
    a, b = fm_eval("bs", opts, n), fm_eval("ld_bs", opts, n)
    fin = np.isfinite(b)
    bad = np.isnan(a) != np.isnan(b)
    assert not bad.any(), (opts[bad][:5], a[bad][:5], b[bad][:5])
    assert np.array_equal(a[~fin & ~np.isnan(b)], b[~fin & ~np.isnan(b)])
    tol = 1e-12 * (opts[fin, 0] + np.abs(b[fin])) + 1e-300
    assert np.all(np.abs(a[fin] - b[fin]) <= tol), np.max(np.abs(a[fin] - b[fin]) / tol)
