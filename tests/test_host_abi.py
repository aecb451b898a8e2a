"""Host-side logic of the C-ABI library (no GPU needed): exports, grid
resolution, generators, arena accounting and launch-time validation — all
against the reference (oracle/_ref) or the oracle."""
import ctypes as C
import subprocess

import numpy as np
import pytest

import oracle
from paper_2308_16877_b200 import abi
from paper_2308_16877_b200 import engine as E


def test_library_exports_every_declared_symbol():
    lib = abi.lib()
    assert lib.hpac_abi_version() == 4
    declared = abi.exported_symbols()
    assert len(declared) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", str(abi.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        getattr(lib, s)


@pytest.mark.ref
@pytest.mark.parametrize("bench", ["blackscholes", "binomial", "kmeans", "synthetic-constant",
                                   "synthetic-slow-drift", "synthetic-noise"])
@pytest.mark.parametrize("n,ov", [(0, {}), (4 * 64 * 20, dict(num_teams=4, items_per_thread=20)),
                                  (1 << 20, dict(items_per_thread=64)), (12345, dict(threads_per_team=32, warp_size=8))])
def test_resolve_grid_matches_reference(ref_lib, bench, n, ov):
    g, mp = E.resolve_grid(bench, n, **ov)
    ovc = abi.Grid(ov.get("num_teams", 0), ov.get("threads_per_team", 0), ov.get("warp_size", 0),
                   ov.get("items_per_thread", 0), 0)
    out = abi.Grid()
    m = C.c_int32()
    assert ref_lib.ref_resolve_grid(bench.encode(), n, C.byref(ovc), C.byref(out), C.byref(m)) == 0
    assert (g.num_teams, g.threads_per_team, g.warp_size, g.items_per_thread, g.shared_mem_budget_bytes) == \
        (out.num_teams, out.threads_per_team, out.warp_size, out.items_per_thread, out.shared_mem_budget_bytes)
    assert mp == m.value


def test_resolve_grid_unknown_benchmark():
    with pytest.raises(E.ConfigError):
        E.resolve_grid("nonesuch")


@pytest.mark.ref
def test_generators_bit_identical_to_reference(ref_lib):
    a = E.make_bs_portfolio(5000, 42)
    b = np.empty_like(a)
    ref_lib.ref_make_bs_portfolio(5000, 42, 512, 0.01, b.ctypes.data)
    assert np.array_equal(a, b)
    a = E.make_binomial_portfolio(5000, 42)
    b = np.empty_like(a)
    ref_lib.ref_make_binomial_portfolio(5000, 42, 0.002, b.ctypes.data)
    assert np.array_equal(a, b)
    a = E.make_blobs(3000, 32, 64, 42, 8.0)
    b = np.empty_like(a)
    ref_lib.ref_make_blobs(3000, 32, 64, 42, 8.0, b.ctypes.data)
    assert np.array_equal(a, b)


def test_portfolios_deterministic_in_seed():
    a = E.make_bs_portfolio(256, 7)
    b = E.make_bs_portfolio(256, 7)
    c = E.make_bs_portfolio(256, 8)
    assert a[100, 0] == b[100, 0]
    assert np.any(a[:, 0] != c[:, 0])


def _region_for(app, in_dims=1, out_dims=1):
    if app == "table":
        x = np.zeros((4, max(in_dims, 1)))
        return E.table_region(x if in_dims else None, np.zeros((4, out_dims)), np.zeros((4, out_dims)),
                              input_dims=in_dims, output_dims=out_dims)
    return E.synthetic_region(0, 1, np.zeros(4))


@pytest.mark.parametrize("spec_fn,tpt,ws,budget", [
    (lambda: E.taf(5, 4, 1.0), 32, 32, 64),        # test_engine.cpp:386-393
    (lambda: E.taf(5, 8, 1.0), 64, 32, 16),        # test_harness.cpp:240-253
    (lambda: E.taf(3, 2, 0.1, "team"), 8, 4, 8 * 40 + 7),
    (lambda: E.iact(4, 0.5), 64, 32, 48 * 1024),
    (lambda: E.iact(8, 0.5, None, "team"), 64, 32, 2 * 32 * 8 * 16 + 2 * 256 + 7),
    (lambda: E.iact(2, 0.5, 4), 64, 32, 100),
])
def test_arena_accounting_matches_oracle(oracle_lib, spec_fn, tpt, ws, budget):
    g = E.GridConfig(1, tpt, ws, 4, budget)
    r = _region_for("table")
    req_o, av_o = C.c_uint64(), C.c_uint64()
    err = C.create_string_buffer(256)
    rc_o = oracle_lib.oracle_arena_required(C.byref(g.c()), C.byref(r.c()), C.byref(spec_fn()),
                                            C.byref(req_o), C.byref(av_o), err, 256)
    try:
        req = E.arena_required(g, r, spec_fn())
        rc = 0
    except E.ArenaOverflowError as e:
        rc, req = 2, e.required_bytes
    assert rc == rc_o
    assert req == req_o.value


@pytest.mark.parametrize("grid,n,msg", [
    (E.GridConfig(0, 32, 32, 1), 1, "num_teams"),
    (E.GridConfig(1, 0, 32, 1), 1, "threads_per_team"),
    (E.GridConfig(1, 32, 65, 1), 1, "warp_size"),
    (E.GridConfig(1, 30, 8, 1), 1, "must divide"),
    (E.GridConfig(1, 32, 32, 0), 1, "items_per_thread"),
    (E.GridConfig(1, 32, 32, 1), 33, "capacity"),
    (E.GridConfig(1, 32, 32, 1), -1, "non-negative"),
])
def test_launch_validation_before_any_device_work(grid, n, msg):
    """ConfigError classes of grid.hpp:27-53 raised host-side (no GPU touched)."""
    with pytest.raises(E.ConfigError, match=msg):
        E.run_region(grid, n, 0, _region_for("synth"), None)


@pytest.mark.parametrize("spec_fn,msg", [
    (lambda: E.taf(0, 1, 0.5), "history size"),
    (lambda: E.taf(1, 0, 0.5), "prediction size"),
    (lambda: E.taf(1, 1, -0.5), "threshold"),
    (lambda: E.iact(0, 0.5), "table size"),
    (lambda: E.iact(1, 0.5, 3), "must divide"),
    (lambda: E.perfo("small", 1), "modulus"),
    (lambda: E.perfo("ini", 0), "percent"),
    (lambda: E.perfo("fini", 100), "percent"),
])
def test_spec_validation(spec_fn, msg):
    with pytest.raises(E.ConfigError, match=msg):
        E.run_region(E.GridConfig(1, 32, 32, 1), 4, 0, _region_for("table"), spec_fn())


def test_iact_needs_inputs():
    with pytest.raises(E.ConfigError, match="inputs"):
        E.run_region(E.GridConfig(1, 32, 32, 1), 4, 0, _region_for("table", in_dims=0), E.iact(2, 0.5))


def test_ini_fini_rejects_encounters():
    x = np.zeros((4, 1))
    r = E.table_region(x, x.copy(), x.copy(), encounters=np.ones(4, np.int32))
    with pytest.raises(E.ConfigError, match="trip count"):
        E.run_region(E.GridConfig(1, 32, 32, 1), 4, 0, r, E.perfo("ini", 50))
