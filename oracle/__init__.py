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

def _load_abi():
    """The ctypes struct layouts of include/hpac_offload.h (abi.py), loaded by
    file path so that importing the checker never imports the product
    package or maps its library (the reference arm of bench.py relies on it)."""
    import importlib.util
    import sys
    name = "paper_2308_16877_b200.abi"
    if name in sys.modules:
        return sys.modules[name]
    path = Path(__file__).resolve().parent.parent / "paper_2308_16877_b200" / "abi.py"
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    # registered under its own name: a later import of the package reuses this
    # module, so both sides share one set of struct classes
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


abi = _load_abi()

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
        L.oracle_run_region_teams.restype = C.c_int
        L.oracle_run_region_teams.argtypes = [P(abi.Grid), C.c_int64, C.c_int32, P(abi.Region), P(abi.Spec),
                                              P(abi.Stats), C.c_void_p, C.c_int32, C.c_int32, C.c_char_p,
                                              C.c_size_t]
        L.oracle_make_lavamd.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_void_p]
        L.oracle_bs_prices.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.oracle_binomial_prices.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p]
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
        L.ref_bench_binomial_run.argtypes = [C.c_void_p, C.c_int64, C.c_int, P(abi.Grid), P(abi.Spec),
                                             C.c_void_p, P(abi.Stats), C.c_char_p, C.c_size_t]
        L.ref_bench_blackscholes_run.argtypes = [C.c_void_p, C.c_int64, P(abi.Grid), P(abi.Spec),
                                                 C.c_void_p, P(abi.Stats), C.c_char_p, C.c_size_t]
        L.ref_binomial_reference.restype = None
        L.ref_binomial_reference.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        L.ref_blackscholes_reference.restype = None
        L.ref_blackscholes_reference.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
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
    grid = grid if isinstance(grid, abi.Grid) else grid.c()
    region = region if isinstance(region, abi.Region) else region.c()
    rc = lib_fn(C.byref(grid), n, mapping, C.byref(region),
                C.byref(spec) if spec is not None else None, C.byref(st),
                paths.ctypes.data if paths is not None else None, err, 1024)
    return rc, st, err.value.decode(errors="replace")


def ref_parse(text):
    """The reference's parse_directive (directive.hpp:522) -> hpac_spec_t."""
    sp = abi.Spec()
    code, off = C.c_int32(), C.c_int64()
    err = C.create_string_buffer(512)
    rc = ref().ref_parse_directive(text.encode(), C.byref(sp), C.byref(code), C.byref(off), err, 512)
    if rc:
        raise ValueError(f"{text!r}: {err.value.decode()}")
    return sp


def ref_grid(benchmark, n, **overrides):
    """The reference's resolve_grid (bench/run.hpp:81-97) -> (hpac_grid_t, mapping)."""
    ov = abi.Grid(overrides.get("num_teams", 0), overrides.get("threads_per_team", 0),
                  overrides.get("warp_size", 0), overrides.get("items_per_thread", 0),
                  overrides.get("shared_mem_budget_bytes", 0))
    g = abi.Grid()
    mp = C.c_int32()
    if ref().ref_resolve_grid(benchmark.encode(), n, C.byref(ov), C.byref(g), C.byref(mp)):
        raise ValueError(f"resolve_grid({benchmark!r}, {n})")
    return g, mp.value


def ref_portfolio(kind, n, seed):
    """The reference's generators: make_binomial_portfolio / make_bs_portfolio."""
    out = np.empty((n, 5))
    if kind == "binomial":
        ref().ref_make_binomial_portfolio(n, seed, 0.002, out.ctypes.data)
    else:
        ref().ref_make_bs_portfolio(n, seed, 512, 0.01, out.ctypes.data)
    return out


def ref_bench_binomial(options, n_steps, grid, spec):
    """bench::binomial_region through the reference's run_region (per team).
    Returns (status, Stats, prices, message)."""
    o = np.ascontiguousarray(options, dtype=np.float64)
    prices = np.zeros(len(o))
    st = abi.Stats()
    err = C.create_string_buffer(512)
    rc = ref().ref_bench_binomial_run(o.ctypes.data, len(o), n_steps, C.byref(grid),
                                      C.byref(spec) if spec is not None else None, prices.ctypes.data,
                                      C.byref(st), err, 512)
    return rc, st, prices, err.value.decode(errors="replace")


def ref_bench_blackscholes(options, grid, spec):
    o = np.ascontiguousarray(options, dtype=np.float64)
    prices = np.zeros(len(o))
    st = abi.Stats()
    err = C.create_string_buffer(512)
    rc = ref().ref_bench_blackscholes_run(o.ctypes.data, len(o), C.byref(grid),
                                          C.byref(spec) if spec is not None else None, prices.ctypes.data,
                                          C.byref(st), err, 512)
    return rc, st, prices, err.value.decode(errors="replace")


def oracle_run(grid, n, mapping, region, spec=None, paths=None):
    return run_region(oracle().oracle_run_region, grid, n, mapping, region, spec, paths)


def ref_run(grid, n, mapping, region, spec=None, paths=None):
    return run_region(ref().ref_run_region, grid, n, mapping, region, spec, paths)


def oracle_run_teams(grid, n, mapping, region, spec, team_range, paths=None):
    """Teams [b, e) of the logical grid only (each keeps its global thread ids
    and stride), the counterpart of hpac_launch_t.team_begin/team_end."""
    st = abi.Stats()
    err = C.create_string_buffer(1024)
    rc = oracle().oracle_run_region_teams(C.byref(grid.c()), n, mapping, C.byref(region.c()),
                                          C.byref(spec) if spec is not None else None, C.byref(st),
                                          paths.ctypes.data if paths is not None else None,
                                          int(team_range[0]), int(team_range[1]), err, 1024)
    return rc, st, err.value.decode(errors="replace")


def make_lavamd(b1, particles, seed):
    n = b1 ** 3 * particles
    rv, qv = np.empty((n, 4)), np.empty(n)
    if oracle().oracle_make_lavamd(b1, particles, seed, rv.ctypes.data, qv.ctypes.data):
        raise ValueError("make_lavamd: bad arguments")
    return rv, qv


def ref_blobs(n, dims, k, seed, separation):
    """The reference's make_blobs (bench/kmeans.hpp:25-47)."""
    out = np.empty((n, dims))
    ref().ref_make_blobs(n, dims, k, seed, separation, out.ctypes.data)
    return out


def bs_prices(options):
    """black_scholes_call per option (NaN where it rejects the option)."""
    o = np.ascontiguousarray(options, dtype=np.float64)
    out = np.empty(len(o))
    oracle().oracle_bs_prices(o.ctypes.data, len(o), out.ctypes.data)
    return out


def binomial_prices(options, steps, american=True, put=True):
    """binomial_price per option (NaN where it rejects the option); all host threads."""
    o = np.ascontiguousarray(options, dtype=np.float64)
    out = np.empty(len(o))
    oracle().oracle_binomial_prices(o.ctypes.data, len(o), steps, int(american), int(put), out.ctypes.data)
    return out


def ref_binomial_prices(options, steps, american=True, put=True, threads=None):
    """The reference's own binomial_price (bench/binomial.hpp:16-50) per
    option, fanned out over host threads (ctypes releases the GIL)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    L = ref()
    o = np.ascontiguousarray(options, dtype=np.float64)
    out = np.empty(len(o))

    def one(i):
        v = C.c_double()
        rc = L.ref_binomial_price(o[i].ctypes.data, steps, int(american), int(put), C.byref(v))
        out[i] = v.value if rc == 0 else np.nan

    with ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1) as ex:
        list(ex.map(one, range(len(o))))
    return out


def ref_bs_prices(options):
    """The reference's own black_scholes_call (bench/blackscholes.hpp:25-36)."""
    L = ref()
    o = np.ascontiguousarray(options, dtype=np.float64)
    out = np.empty(len(o))
    v = C.c_double()
    for i in range(len(o)):
        rc = L.ref_black_scholes_call(o[i].ctypes.data, C.byref(v))
        out[i] = v.value if rc == 0 else np.nan
    return out
