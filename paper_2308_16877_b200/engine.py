"""Python host mirror of the reference's approximate-region API.

Names and argument meaning follow simtac (paths relative to
/root/reference/proj/include/simtac/):

* ``GridConfig``            <- grid.hpp:16-54 (same defaults)
* ``WorkMapping``           <- grid.hpp:14
* ``ApproxSpec`` helpers     <- directive.hpp:59-84 (``taf``, ``iact``, ``perfo``)
* Regions                    <- engine.hpp:26-33 and bench/*.hpp region builders
* ``run_region``            <- engine.hpp:132-134, returns ``LaunchResult``
                               (engine.hpp:35-54)
* exceptions                 <- errors.hpp:12-62 (+ DirectiveError, directive.hpp:120)

Every call goes through the C-ABI (libhpac_b200.so) onto the GPU; buffers
are torch CUDA tensors (device) or numpy arrays for ``run_region_host``.
There is no CPU execution path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import abi

# ---- errors (errors.hpp) ---------------------------------------------------


class SimtError(RuntimeError):
    pass


class ConfigError(SimtError):
    pass


class ArenaOverflowError(SimtError):
    def __init__(self, msg, required=0, available=0):
        super().__init__(msg)
        self.required_bytes = required
        self.available_bytes = available


class BarrierDivergenceError(SimtError):
    def __init__(self, msg, team=0, step=0, missing=0):
        super().__init__(msg)
        self.team_id = team
        self.step = step
        self.missing = missing


class DirectiveError(SimtError):
    def __init__(self, msg, code=-1, offset=-1):
        super().__init__(msg)
        self.code = code
        self.offset = offset


class UnsupportedError(SimtError):
    pass


class CudaError(SimtError):
    pass


def _raise(rc, err, stats=None):
    msg = err.value.decode(errors="replace") if hasattr(err, "value") else str(err)
    if rc == abi.ERR_CONFIG:
        raise ConfigError(msg)
    if rc == abi.ERR_ARENA_OVERFLOW:
        raise ArenaOverflowError(msg, stats.arena_required if stats else 0,
                                 stats.arena_available if stats else 0)
    if rc == abi.ERR_BARRIER_DIVERGENCE:
        raise BarrierDivergenceError(msg, stats.fail_team, stats.fail_step, stats.fail_missing)
    if rc == abi.ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if rc == abi.ERR_CUDA:
        raise CudaError(msg)
    raise SimtError(f"status {rc}: {msg}")


# ---- grid / mapping --------------------------------------------------------

class WorkMapping:
    PER_THREAD = abi.MAP_PER_THREAD
    PER_TEAM = abi.MAP_PER_TEAM


@dataclass
class GridConfig:
    num_teams: int = 1
    threads_per_team: int = 32
    warp_size: int = 32
    items_per_thread: int = 1
    shared_mem_budget_bytes: int = 48 * 1024

    def c(self):
        return abi.Grid(self.num_teams, self.threads_per_team, self.warp_size,
                        self.items_per_thread, self.shared_mem_budget_bytes)

    def total_threads(self):
        return self.num_teams * self.threads_per_team


def resolve_grid(benchmark: str, n: int = 0, **overrides):
    """bench::resolve_grid (bench/run.hpp:81-97); returns (GridConfig, mapping)."""
    ov = abi.Grid(overrides.get("num_teams", 0), overrides.get("threads_per_team", 0),
                  overrides.get("warp_size", 0), overrides.get("items_per_thread", 0),
                  overrides.get("shared_mem_budget_bytes", 0))
    out = abi.Grid()
    mp = C.c_int32()
    err = C.create_string_buffer(512)
    rc = abi.lib().hpac_resolve_grid(benchmark.encode(), n, C.byref(ov), C.byref(out),
                                     C.byref(mp), err, 512)
    if rc:
        _raise(rc, err)
    return GridConfig(out.num_teams, out.threads_per_team, out.warp_size, out.items_per_thread,
                      out.shared_mem_budget_bytes), mp.value


# ---- spec ------------------------------------------------------------------

def taf(h_size, p_size, threshold, level="thread"):
    """memo(out:h:p:thr) — TafConfig, taf.hpp:14-25."""
    s = abi.Spec()
    s.technique = abi.TECH_TAF
    s.level = abi.LEVELS[level] if isinstance(level, str) else level
    s.taf_h_size, s.taf_p_size, s.taf_threshold = h_size, p_size, float(threshold)
    s.n_output_sections = 1
    return s


def iact(table_size, threshold, tables_per_warp=None, level="thread"):
    """memo(in:size:thr[:tpw]) — IactConfig, iact.hpp:16-41."""
    s = abi.Spec()
    s.technique = abi.TECH_IACT
    s.level = abi.LEVELS[level] if isinstance(level, str) else level
    s.iact_table_size, s.iact_threshold = table_size, float(threshold)
    s.iact_tables_per_warp = 0 if tables_per_warp is None else tables_per_warp
    s.n_input_sections = 1
    s.n_output_sections = 1
    return s


def perfo(kind, arg, level="thread", seed=0):
    """perfo(kind:arg) — PerfoConfig, perfo.hpp:22-36 (+ random extension)."""
    s = abi.Spec()
    s.technique = abi.TECH_PERFO
    s.level = abi.LEVELS[level] if isinstance(level, str) else level
    s.perfo_kind = abi.PERFO_KINDS[kind] if isinstance(kind, str) else kind
    if s.perfo_kind in (abi.PERFO_INI, abi.PERFO_FINI, abi.PERFO_RANDOM):
        s.perfo_skip_percent = arg
    else:
        s.perfo_modulus = arg
    s.perfo_seed = seed
    return s


def parse_directive(text: str):
    """parse_directive (directive.hpp:522) -> (Spec, canonical text)."""
    spec = abi.Spec()
    code = C.c_int32(-1)
    off = C.c_int64(-1)
    err = C.create_string_buffer(1024)
    rc = abi.lib().hpac_parse_directive(text.encode(), C.byref(spec), C.byref(code),
                                        C.byref(off), err, 1024)
    if rc == abi.ERR_DIRECTIVE:
        raise DirectiveError(err.value.decode(), code.value, off.value)
    if rc:
        _raise(rc, err)
    return spec, err.value.decode()


def unparse(spec) -> str:
    buf = C.create_string_buffer(1024)
    rc = abi.lib().hpac_unparse(C.byref(spec), buf, 1024)
    if rc:
        _raise(rc, buf)
    return buf.value.decode()


# ---- regions ---------------------------------------------------------------

def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


@dataclass
class Region:
    """Region descriptor (engine.hpp:26-33): app id + caller-owned buffers."""
    app: int
    input_dims: int = 0
    output_dims: int = 1
    flags: int = 0
    synthetic_profile: int = 0
    binomial_steps: int = 32
    binomial_american: int = 1
    binomial_put: int = 1
    kmeans_dims: int = 2
    kmeans_k: int = 8
    lavamd_boxes1d: int = 0
    lavamd_particles: int = 0
    lavamd_alpha: float = 0.5
    seed: int = 0
    inputs: object = None
    table_out: object = None
    encounters: object = None
    out: object = None
    centroids: object = None
    labels: object = None

    def c(self):
        r = abi.Region()
        r.app, r.input_dims, r.output_dims, r.flags = self.app, self.input_dims, self.output_dims, self.flags
        r.synthetic_profile, r.binomial_steps = self.synthetic_profile, self.binomial_steps
        r.binomial_american, r.binomial_put = self.binomial_american, self.binomial_put
        r.kmeans_dims, r.kmeans_k, r.seed = self.kmeans_dims, self.kmeans_k, self.seed
        r.lavamd_boxes1d, r.lavamd_particles = self.lavamd_boxes1d, self.lavamd_particles
        r.lavamd_alpha = self.lavamd_alpha
        r.in_ = _ptr(self.inputs)
        r.table_out = _ptr(self.table_out)
        r.encounters = _ptr(self.encounters)
        r.out = _ptr(self.out)
        r.centroids = _ptr(self.centroids)
        r.labels = _ptr(self.labels)
        return r


def table_region(inputs, table_out, out, input_dims=None, output_dims=None, encounters=None,
                 accumulate=False, barrier=False):
    """A pure region given by its accurate outputs per work item."""
    in_dims = input_dims if input_dims is not None else (0 if inputs is None else
                                                        (inputs.shape[1] if inputs.ndim > 1 else 1))
    out_dims = output_dims if output_dims is not None else (table_out.shape[1] if table_out.ndim > 1 else 1)
    flags = (abi.REGION_STORE_ACCUMULATE if accumulate else 0) | (abi.REGION_BARRIER_IN_EVALUATE if barrier else 0)
    return Region(abi.APP_TABLE, in_dims, out_dims, flags, inputs=inputs, table_out=table_out,
                  encounters=encounters, out=out)


def synthetic_region(profile, seed, out):
    """bench::synthetic_region (bench/synthetic.hpp:56-71)."""
    return Region(abi.APP_SYNTHETIC, 1, 1, synthetic_profile=profile, seed=seed, out=out)


def blackscholes_region(options, prices):
    """bench::blackscholes_region (bench/blackscholes.hpp:72-92); options n x 5."""
    return Region(abi.APP_BLACKSCHOLES, 5, 1, inputs=options, out=prices)


def binomial_region(options, n_steps, prices, american=True, put=True):
    """bench::binomial_region (bench/binomial.hpp:74-94)."""
    return Region(abi.APP_BINOMIAL, 5, 1, binomial_steps=n_steps, binomial_american=int(american),
                  binomial_put=int(put), inputs=options, out=prices)


def kmeans_region(points, centroids, labels, distances=None, fast_math=False):
    """Distance region of kmeans_benchmark (bench/kmeans.hpp:82-102) + fused argmin."""
    n, d = points.shape
    k = centroids.shape[0]
    return Region(abi.APP_KMEANS, d, k, abi.REGION_KMEANS_FAST_MATH if fast_math else 0,
                  kmeans_dims=d, kmeans_k=k, inputs=points, centroids=centroids, labels=labels,
                  out=distances)


def lavamd_region(rv, qv, fv, boxes1d, particles, alpha=0.5):
    """LavaMD (Rodinia lavaMD restated): item = home box,
    lane = home particle, encounter = neighbour box; fv accumulates."""
    return Region(abi.APP_LAVAMD, 0, 4, lavamd_boxes1d=boxes1d, lavamd_particles=particles,
                  lavamd_alpha=alpha, inputs=rv, table_out=qv, out=fv)


def make_lavamd(boxes1d, particles, seed):
    n = boxes1d ** 3 * particles
    rv = np.empty((n, 4))
    qv = np.empty(n)
    if abi.lib().hpac_make_lavamd(boxes1d, particles, seed, rv.ctypes.data, qv.ctypes.data):
        raise ConfigError("make_lavamd: bad arguments")
    return rv, qv


# ---- launch ----------------------------------------------------------------

@dataclass
class LaunchResult:
    stats: dict = field(default_factory=dict)
    kernel_ms: float = 0.0

    def approx_rate(self):
        t = self.stats["total_invocations"]
        return 0.0 if t == 0 else self.stats["approx_invocations"] / t

    def divergent_fraction(self):
        t = self.stats["total_warp_steps"]
        return 0.0 if t == 0 else self.stats["divergent_warp_steps"] / t


def run_region(grid: GridConfig, n: int, mapping: int, region: Region, spec=None, *, stream=None,
               paths=None, team_range=None, synchronous=True) -> LaunchResult:
    """run_region on the device (engine.hpp:132). Buffers: torch CUDA tensors."""
    st = abi.Stats()
    L = abi.Launch()
    L.stream = stream if isinstance(stream, int) else (stream.cuda_stream if stream is not None else None)
    if team_range is not None:
        L.team_begin, L.team_end = team_range
    L.paths = _ptr(paths)
    L.synchronous = 1 if synchronous else 0
    err = C.create_string_buffer(1024)
    rc = abi.lib().hpac_run_region(C.byref(grid.c()), n, mapping, C.byref(region.c()),
                                   C.byref(spec) if spec is not None else None, C.byref(L),
                                   C.byref(st), err, 1024)
    if rc:
        _raise(rc, err, st)
    return LaunchResult(st.as_dict(), st.kernel_ms)


def run_region_host(grid: GridConfig, n: int, mapping: int, region: Region, spec=None,
                    team_range=None) -> LaunchResult:
    """Same call with host (numpy) buffers: H2D, run, D2H inside. team_range =
    (begin, end): only those logical teams run, and only their items move
    (hpac_run_region_host_teams; Blackscholes and Binomial)."""
    st = abi.Stats()
    err = C.create_string_buffer(1024)
    if team_range is not None:
        rc = abi.lib().hpac_run_region_host_teams(C.byref(grid.c()), n, mapping, C.byref(region.c()),
                                                  C.byref(spec) if spec is not None else None,
                                                  int(team_range[0]), int(team_range[1]),
                                                  C.byref(st), err, 1024)
    else:
        rc = abi.lib().hpac_run_region_host(C.byref(grid.c()), n, mapping, C.byref(region.c()),
                                            C.byref(spec) if spec is not None else None,
                                            C.byref(st), err, 1024)
    if rc:
        _raise(rc, err, st)
    return LaunchResult(st.as_dict(), st.kernel_ms)


def arena_required(grid: GridConfig, region: Region, spec):
    req, avail = C.c_uint64(), C.c_uint64()
    err = C.create_string_buffer(512)
    rc = abi.lib().hpac_arena_required(C.byref(grid.c()), C.byref(region.c()), C.byref(spec),
                                       C.byref(req), C.byref(avail), err, 512)
    if rc == abi.ERR_ARENA_OVERFLOW:
        raise ArenaOverflowError(err.value.decode(), req.value, avail.value)
    if rc:
        _raise(rc, err)
    return req.value


# ---- K-Means Lloyd loop -----------------------------------------------------

@dataclass
class KmeansResult:
    assignments: object
    centroids: object
    iterations: int
    converged: bool
    stats: dict
    region_ms: float
    update_ms: float
    graph: bool = False  # the iterations ran as one CUDA graph launch


def kmeans_run(grid: GridConfig, points, k, spec=None, max_iters=40, centroids=None,
               fast_math=False, perfo_seed_base=0, allreduce=None, stream=None,
               nccl_comm=None, host_loop=False) -> KmeansResult:
    """kmeans_benchmark (bench/kmeans.hpp:62-144) on the device. `points` is a
    torch CUDA tensor n x d. `allreduce(buf_tensor)` (optional) all-reduces the
    packed [sums | counts | changed] partials across ranks each iteration;
    `nccl_comm` (an ncclComm_t handle) uses the library's native NCCL hook
    (hpac_nccl_allreduce) instead. Without a hook the loop runs as one CUDA
    graph launch (device-side convergence); host_loop=True forces one
    synchronised host round trip per iteration."""
    import torch
    n, d = points.shape
    cent = torch.empty((k, d), dtype=torch.float64, device=points.device) if centroids is None else centroids
    assign = torch.empty(n, dtype=torch.int32, device=points.device)
    red = torch.empty(k * d + k + 1, dtype=torch.float64, device=points.device)
    pb = abi.KmeansProblem()
    pb.n_points, pb.dims, pb.k = n, d, k
    pb.points, pb.centroids, pb.assignments = _ptr(points), _ptr(cent), _ptr(assign)
    pb.max_iters = max_iters
    pb.flags = (abi.REGION_KMEANS_FAST_MATH if fast_math else 0) | \
        (abi.KMEANS_CENTROIDS_GIVEN if centroids is not None else 0) | \
        (abi.KMEANS_HOST_LOOP if host_loop else 0)
    pb.perfo_seed_base = perfo_seed_base
    pb.reduce_buf = _ptr(red)
    cb = None
    hook_error = []
    if nccl_comm is not None:
        pb.allreduce = C.cast(abi.lib().hpac_nccl_allreduce, abi.ALLREDUCE_FN)
        pb.allreduce_user = nccl_comm
    elif allreduce is not None:
        def _cb(buf, count, user, st):
            # The library produced `red` on stream `st` and reads it back there,
            # while torch orders the collective against its current stream:
            # when the two differ, torch's stream waits for `st` before the
            # all-reduce and `st` waits for torch's stream after it. An
            # exception cannot cross the C boundary, so it is kept, reported as
            # a nonzero status (the loop stops with HPAC_ERR_CUDA) and
            # re-raised below.
            try:
                cur = torch.cuda.current_stream(points.device)
                lib_stream = torch.cuda.ExternalStream(st, device=points.device) \
                    if st and st != cur.cuda_stream else None
                if lib_stream is not None:
                    cur.wait_stream(lib_stream)
                allreduce(red)
                if lib_stream is not None:
                    lib_stream.wait_stream(cur)
                return 0
            except BaseException as exc:  # noqa: BLE001 - re-raised after the run
                hook_error.append(exc)
                return 1
        cb = abi.ALLREDUCE_FN(_cb)
        pb.allreduce = cb
    res = abi.KmeansResult()
    err = C.create_string_buffer(1024)
    st = stream if isinstance(stream, int) else (stream.cuda_stream if stream is not None else None)
    rc = abi.lib().hpac_kmeans_run(C.byref(grid.c()), C.byref(pb),
                                   C.byref(spec) if spec is not None else None, st,
                                   C.byref(res), err, 1024)
    if hook_error:
        raise CudaError(f"kmeans all-reduce hook failed: {hook_error[0]!r}") from hook_error[0]
    if rc:
        _raise(rc, err, res.stats)
    return KmeansResult(assign, cent, res.iterations, bool(res.converged), res.stats.as_dict(),
                        res.region_ms, res.update_ms, bool(res.graph))


def nccl_comms(ndev=1):
    """Single-process NCCL communicators over devices 0..ndev-1 (ncclCommInitAll)."""
    comms = (C.c_void_p * ndev)()
    devs = (C.c_int * ndev)(*range(ndev))
    rc = abi.lib().hpac_nccl_comm_init_all(ndev, devs, comms)
    if rc:
        raise UnsupportedError("NCCL unavailable") if rc == abi.ERR_UNSUPPORTED else CudaError("ncclCommInitAll")
    return list(comms)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0), to broadcast to the other ranks."""
    buf = C.create_string_buffer(128)
    rc = abi.lib().hpac_nccl_unique_id(buf)
    if rc:
        raise UnsupportedError("NCCL unavailable") if rc == abi.ERR_UNSUPPORTED else CudaError("ncclGetUniqueId")
    return buf.raw


def nccl_comm_init_rank(nranks: int, uid: bytes, rank: int):
    """Join a multi-process NCCL communicator (one process per GPU); the
    handle is kmeans_run's `nccl_comm`."""
    comm = C.c_void_p()
    rc = abi.lib().hpac_nccl_comm_init_rank(nranks, uid, rank, C.byref(comm))
    if rc:
        raise UnsupportedError("NCCL unavailable") if rc == abi.ERR_UNSUPPORTED else CudaError("ncclCommInitRank")
    return comm.value


# ---- generators (host) -----------------------------------------------------

def make_bs_portfolio(n, seed, base_block=512, jitter=0.01):
    out = np.empty((n, 5), dtype=np.float64)
    if abi.lib().hpac_make_bs_portfolio(n, seed, base_block, jitter, out.ctypes.data):
        raise ConfigError("make_bs_portfolio: bad arguments")
    return out


def make_binomial_portfolio(n, seed, jitter=0.002):
    out = np.empty((n, 5), dtype=np.float64)
    if abi.lib().hpac_make_binomial_portfolio(n, seed, jitter, out.ctypes.data):
        raise ConfigError("make_binomial_portfolio: bad arguments")
    return out


def make_blobs(n, dims, k, seed, separation=6.0):
    out = np.empty((n, dims), dtype=np.float64)
    if abi.lib().hpac_make_blobs(n, dims, k, seed, separation, out.ctypes.data):
        raise ConfigError("make_blobs: bad arguments")
    return out


def mape(accurate, approximate, stream=None):
    r = C.c_double()
    rc = abi.lib().hpac_mape(_ptr(accurate), _ptr(approximate), accurate.numel(), stream, C.byref(r))
    if rc:
        raise CudaError("mape failed")
    return r.value


def mcr(accurate, approximate, stream=None):
    r = C.c_double()
    rc = abi.lib().hpac_mcr(_ptr(accurate), _ptr(approximate), accurate.numel(), stream, C.byref(r))
    if rc:
        raise CudaError("mcr failed")
    return r.value
