"""TEST INFRASTRUCTURE ONLY — CPU checker for the CUDA path.

Python bindings to
  * oracle/liboracle.so          — C restatement of the reference engine (hpac_oracle.c)
  * oracle/_ref/libsimtac_ref.so — the reference itself, compiled from
                                   /root/reference/proj/include (ref_shim.cpp)
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2308_16877_b200 import abi

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libsimtac_ref.so"
REF_ROOT = Path("/root/reference/proj/include")

P = C.POINTER


def build(ref: bool = True):
    """Compile the checker (and the reference, when its sources are present)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if ref and REF_ROOT.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


_cache = {}


def _run_sig(f):
    f.restype = C.c_int
    f.argtypes = [P(abi.Grid), C.c_int64, C.c_int32, P(abi.Region), P(abi.Spec), P(abi.Stats),
                  C.c_void_p, C.c_char_p, C.c_size_t]


def oracle():
    if "o" not in _cache:
        if not ORACLE_SO.exists():
            build(ref=False)
        L = C.CDLL(str(ORACLE_SO))
        _run_sig(L.oracle_run_region)
        L.oracle_black_scholes_call.argtypes = [C.c_void_p, P(C.c_double)]
        L.oracle_binomial_price.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, P(C.c_double)]
        L.oracle_synthetic_value.restype = C.c_double
        L.oracle_synthetic_value.argtypes = [C.c_int, C.c_int64, C.c_uint64]
        L.oracle_rsd.restype = C.c_double
        L.oracle_rsd.argtypes = [C.c_void_p, C.c_int]
        L.oracle_taf_drive.restype = C.c_int64
        L.oracle_taf_drive.argtypes = [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        L.oracle_taf_state_bytes.restype = C.c_uint64
        L.oracle_taf_state_bytes.argtypes = [C.c_int, C.c_int]
        L.oracle_table_group_bytes.restype = C.c_uint64
        L.oracle_table_group_bytes.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        L.oracle_kmeans_benchmark.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, P(abi.Grid), P(abi.Spec), C.c_int, C.c_uint64, C.c_void_p, C.c_void_p, P(C.c_int32), P(C.c_int32), P(abi.Stats), C.c_char_p, C.c_size_t]
        L.oracle_mape.restype = C.c_double
        L.oracle_mape.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.oracle_mcr.restype = C.c_double
        L.oracle_mcr.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.oracle_random_skip.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int]
        L.oracle_arena_required.argtypes = [P(abi.Grid), P(abi.Region), P(abi.Spec), P(C.c_uint64), P(C.c_uint64), C.c_char_p, C.c_size_t]
        _cache["o"] = L
    return _cache["o"]


def ref_available():
    return REF_SO.exists() or REF_ROOT.exists()


def ref():
    if "r" not in _cache:
        if not REF_SO.exists():
            build(ref=True)
        L = C.CDLL(str(REF_SO))
        _run_sig(L.ref_run_region)
        L.ref_black_scholes_call.argtypes = [C.c_void_p, P(C.c_double)]
        L.ref_binomial_price.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, P(C.c_double)]
        L.ref_synthetic_value.restype = C.c_double
        L.ref_synthetic_value.argtypes = [C.c_int, C.c_int64, C.c_uint64]
        L.ref_make_bs_portfolio.argtypes = [C.c_int64, C.c_uint64, C.c_int, C.c_double, C.c_void_p]
        L.ref_make_binomial_portfolio.argtypes = [C.c_int64, C.c_uint64, C.c_double, C.c_void_p]
        L.ref_make_blobs.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_void_p]
        L.ref_kmeans_benchmark.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, P(abi.Grid), P(abi.Spec), C.c_int, C.c_void_p, P(C.c_int32), P(C.c_int32), P(abi.Stats), C.c_char_p, C.c_size_t]
        L.ref_rsd.restype = C.c_double
        L.ref_rsd.argtypes = [C.c_void_p, C.c_int]
        for nm in ("ref_taf_drive", "ref_taf_reference_oracle"):
            f = getattr(L, nm)
            f.restype = C.c_int64
            f.argtypes = [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        L.ref_parse_directive.argtypes = [C.c_char_p, P(abi.Spec), P(C.c_int32), P(C.c_int64), C.c_char_p, C.c_size_t]
        L.ref_resolve_grid.argtypes = [C.c_char_p, C.c_int64, P(abi.Grid), P(abi.Grid), P(C.c_int32)]
        L.ref_mape.restype = C.c_double
        L.ref_mape.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_mcr.restype = C.c_double
        L.ref_mcr.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        _cache["r"] = L
    return _cache["r"]


def _region_np(region):
    """Region whose buffers are numpy arrays (host pointers)."""
    return region.c()


def run_region(lib_fn, grid, n, mapping, region, spec=None, paths=None):
    """Run a region (numpy buffers) through oracle_run_region / ref_run_region.

    Returns (status, Stats, message)."""
    st = abi.Stats()
    err = C.create_string_buffer(1024)
    rc = lib_fn(C.byref(grid.c()), n, mapping, C.byref(region.c()),
                C.byref(spec) if spec is not None else None, C.byref(st),
                paths.ctypes.data if paths is not None else None, err, 1024)
    return rc, st, err.value.decode(errors="replace")


def oracle_run(grid, n, mapping, region, spec=None, paths=None):
    return run_region(oracle().oracle_run_region, grid, n, mapping, region, spec, paths)


def ref_run(grid, n, mapping, region, spec=None, paths=None):
    return run_region(ref().ref_run_region, grid, n, mapping, region, spec, paths)


def bs_prices(options):
    L = oracle()
    out = np.empty(len(options))
    o = np.ascontiguousarray(options, dtype=np.float64)
    v = C.c_double()
    for i in range(len(o)):
        rc = L.oracle_black_scholes_call(o[i].ctypes.data, C.byref(v))
        out[i] = v.value if rc == 0 else np.nan
    return out


def binomial_prices(options, steps, american=True, put=True):
    L = oracle()
    out = np.empty(len(options))
    o = np.ascontiguousarray(options, dtype=np.float64)
    v = C.c_double()
    for i in range(len(o)):
        rc = L.oracle_binomial_price(o[i].ctypes.data, steps, int(american), int(put), C.byref(v))
        out[i] = v.value if rc == 0 else np.nan
    return out
