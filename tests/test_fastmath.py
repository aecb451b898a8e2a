"""csrc/fastmath.cuh on the host (g++ build of the same header): exp/log
within 1 ulp, erfc within 4 ulp (libdevice's documented bounds), IEEE special
values. The device build is checked in test_gpu_fastmath.py."""
import ctypes
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from fastmath_ref import BOUNDS, reference, samples, ulp_errors

ROOT = Path(__file__).resolve().parents[1]
KINDS = {"exp": 0, "log": 1, "erfc": 2, "rcp": 3}


@pytest.fixture(scope="module")
def fm(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ missing")
    so = tmp_path_factory.mktemp("fm") / "libfm_host.so"
    subprocess.run([gxx, "-O2", "-ffp-contract=off", "-shared", "-fPIC",
                    "-I", str(ROOT / "paper_2308_16877_b200" / "csrc"),
                    str(ROOT / "tests" / "cpp" / "fastmath_host.cpp"), "-o", str(so)], check=True)
    lib = ctypes.CDLL(str(so))
    lib.fm_eval_host.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]

    def ev(kind, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        lib.fm_eval_host(KINDS[kind], x.ctypes.data, y.ctypes.data, len(x))
        return y
    return ev


@pytest.mark.parametrize("kind", ["exp", "log", "erfc", "rcp"])
def test_ulp_bound(fm, kind):
    x = samples(kind)
    err = ulp_errors(fm(kind, x), reference(kind, x))
    assert err.max() <= BOUNDS[kind], (kind, err.max(), x[err.argmax()])


def test_special_values(fm):
    nan, inf = np.nan, np.inf
    y = fm("exp", [nan, -inf, inf, -1000.0, 1000.0, 0.0])
    assert np.isnan(y[0]) and list(y[1:]) == [0.0, inf, 0.0, inf, 1.0]
    y = fm("log", [0.0, -1.0, inf, nan, 1.0])
    assert y[0] == -inf and np.isnan(y[1]) and y[2] == inf and np.isnan(y[3]) and y[4] == 0.0
    y = fm("erfc", [nan, -inf, inf, 30.0, -30.0, 0.0, 27.3])
    assert np.isnan(y[0]) and list(y[1:]) == [2.0, 0.0, 0.0, 2.0, 1.0, 0.0]
