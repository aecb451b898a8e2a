#!/usr/bin/env python3
"""Benchmark of the approximate-region hot path (BASELINE.json metric:
"approx-region items/s & speedup vs exact GPU kernel at <=1% quality loss").

Default workload (configs[1]): Binomial options, 1,048,576 American puts x
1024-step CRR lattice under team-shared iACT input memoization
(memo(in:4:0.4) level(team), kPerTeam mapping, 64-thread teams, 384 items
per team — the paper's items-per-thread knob: more options per team table,
more reuse). One step =
one pass of the region over the whole portfolio with inputs resident in
HBM. Per-GPU work is fixed (weak scaling): each rank prices its own
1,048,576-option shard; no collective on the data path.

Prints ONE JSON line on rank 0 (see DESIGN.md §Measurement for every key).
  python bench.py [--gpus N --steps K --warmup W] [--workload binomial|blackscholes|kmeans]
  python bench.py --impl reference ...   # the reference's CPU engine (oracle/_ref)
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "approx-region items/s & speedup vs exact GPU kernel at <=1% quality loss"

# Workload definitions (the N=1 headline is "binomial").
WORKLOADS = {
    "binomial": dict(
        name="binomial-1M-x-1024-iact-team",
        benchmark="binomial", n=1 << 20, lattice=1024, ipt=384, exact_best_ipt=256,
        directive="memo(in:4:0.4) level(team) in(option[i*5:5]) out(price[i])",
        spec=("iact", 4, 0.4, None, "team"),
        unit="options/s"),
    "blackscholes": dict(
        name="blackscholes-4M-taf-h5", benchmark="blackscholes", n=1 << 22, ipt=16,
        directive="memo(out:5:1:0.5) out(price[i])", spec=("taf", 5, 1, 0.5, "thread"), unit="options/s"),
    "lavamd": dict(
        name="lavamd-64^3-boxes-x-128-taf-warp", benchmark="lavamd", boxes1d=64, particles=128, ipt=1,
        directive="memo(out:3:8:0.1) level(warp) out(fv[i*4:4])", spec=("taf", 3, 8, 0.1, "warp"),
        compare_levels=("thread", "team"), unit="particles/s"),
    # C3 as the reference's kmeans_benchmark (bench/kmeans.hpp:62-144): the
    # whole Lloyd loop (region + centroid update + per-iteration all-reduce),
    # to convergence or 40 iterations; one step = one full run
    "kmeans": dict(
        name="kmeans-lloyd-16M-x-32-x-64-perfo-random-team", benchmark="kmeans_lloyd", n=1 << 24,
        dims=32, k=64, ipt=4, separation=30.0, max_iters=40,
        directive="perfo(random:52) level(team)", spec=("perfo", "random", 52, "team"),
        unit="point-iterations/s"),
    # one distance-region launch with a reference perforation kind
    "kmeans-region": dict(
        name="kmeans-16M-x-32-x-64-perfo-small", benchmark="kmeans", n=1 << 24, dims=32, k=64,
        ipt=4, directive="perfo(small:2)", spec=("perfo", "small", 2), unit="point-iterations/s"),
}

# Algorithmic work per item: binomial lattice FP64 flops
# per evaluated option = 5 per node x N(N+1)/2 nodes.
def lava_neighbour_counts(boxes, b1):
    """Neighbour boxes (incl. self) of each home box in a b1^3 grid."""
    import numpy as np
    b = np.asarray(boxes)
    c = np.ones_like(b)
    for coord in (b % b1, (b // b1) % b1, b // (b1 * b1)):
        c = c * (3 - (coord == 0) - (coord == b1 - 1))
    return c


def lava_cpu_scale(m, b1):
    """Boxes 0..m-1 sit on the grid boundary (fewer neighbours): factor that
    converts their particle rate to the b1^3 system's average work/particle."""
    import numpy as np
    sample = lava_neighbour_counts(np.arange(m), b1).mean()
    full = ((2 * 2 + (b1 - 2) * 3) / b1) ** 3
    return sample / full


def binomial_flops(N):
    return 5.0 * N * (N + 1) / 2.0


FP64_PEAK_SOURCE = "in-run DFMA probe (hpac_probe_fp64_peak); MEASURED_PEAKS.json has no FP64 figure"
DMMA_PEAK_SOURCE = ("in-run FP64 tensor-op probe (hpac_probe_dmma_peak, mma.sync m8n8k4 f64); "
                    "MEASURED_PEAKS.json has no FP64 figure")


def lloyd_launches(r, dmma, random_first_exact):
    """Kernels one hpac_kmeans_run launches (kmeans.cu): the label init; per
    host-driven iteration the region (+ its DMMA operand kernel), the label
    compaction, the update partials, their reduction, and - unless that
    iteration converged - accumulate + recompute; in the CUDA graph, a state
    init and per iteration those seven plus three timing/condition kernels
    (accumulate/recompute always run there and return early on convergence)."""
    region = 2 if dmma else 1
    per_host = region + 3 + 2
    it, host_its = r.iterations, r.iterations
    n = 1
    if r.graph:
        host_its = 1 if random_first_exact else 0
        n += 1 + (it - host_its) * (per_host + 3)
    n += host_its * per_host
    if r.converged and not r.graph:
        n -= 2
    return n


def kmeans_uses_dmma(d, k):
    """The runtime's gate for AppKmeansDmma (runtime.cu prepare): 32 dims,
    k % 8 == 0, labels only, whole hardware warps (tpt 64)."""
    return d == 32 and k % 8 == 0


def kmeans_flops(d, k):
    return 3.0 * d * k + k  # sub, mul, add per (c, d) + sqrt per centroid


def kmeans_filter_flops(d, k):
    # executed filter (apps.cuh AppKmeans::eval): x.c as one DFMA per (c, d),
    # |x|^2 (d DFMA), per centroid |x|^2+|c|^2, -2 dot, compare: 2dk + 2d + 3k
    return 2.0 * d * k + 2.0 * d + 3.0 * k


# LavaMD pair term: SURVEY §8(d)'s algorithmic ~40 FP64 flops per particle
# pair (Rodinia's pair term with its exp); our restatement executes 45.3
LAVAMD_PAIR_FLOPS = 40.0  # ~40 per pair (Rodinia pair term with exp); executed: 45.3 (profiles/r03_lavamd_flops.txt)


# ------------------------------------------------------------------ helpers

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def gpu_index(local):
    """LOCAL_RANK -> device. BENCH_DIST_BACKEND=gloo (multi-rank logic check on
    a box with fewer GPUs than ranks) wraps ranks onto the available GPUs."""
    import torch
    if os.environ.get("BENCH_DIST_BACKEND", "nccl") == "gloo":
        return local % max(1, torch.cuda.device_count())
    return local


def init_dist(ws, local):
    """One process per GPU: NCCL process group (barriers, max-over-ranks
    timing, the K-Means all-reduce); BENCH_DIST_BACKEND=gloo for the
    single-GPU check of the N>1 code path."""
    if ws <= 1:
        return None
    import torch
    import torch.distributed as dist
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return dist


def load_traffic(workload):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(workload)
        except Exception:
            return None
    return None


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {}


def make_spec(E, s):
    if s[0] == "iact":
        return E.iact(s[1], s[2], s[3], s[4])
    if s[0] == "taf":
        return E.taf(s[1], s[2], s[3], s[4])
    return E.perfo(s[1], s[2], level=s[3] if len(s) > 3 else "thread")


# ------------------------------------------------------------------ shared config

def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def global_problem(wl, ws):
    """Items of the whole job and how ranks split them. Binomial (the
    headline): ONE logical grid over ws x 2^20 options, split into contiguous
    team ranges that keep the global stride (machine.hpp:77-84), so every
    rank makes exactly the decisions the 1-GPU run of the same problem makes
    (SURVEY §8e). Other workloads: independent per-rank shards."""
    if wl["benchmark"] == "binomial":
        return ws * wl["n"], "team-ranges"
    return wl.get("n"), "shards"


def bench_config(wl, grid, mapping, ws):
    """The `config` object of both arms (identical keys and values)."""
    n_total, split = global_problem(wl, ws)
    per_item = wl.get("particles", 1) if wl["benchmark"] == "lavamd" else 1
    cfg = {"workload": wl["name"], "directive": wl["directive"],
           "grid": {"num_teams": grid.num_teams, "threads_per_team": grid.threads_per_team,
                    "warp_size": grid.warp_size, "items_per_thread": grid.items_per_thread},
           "mapping": "per-team" if mapping == 1 else "per-thread",
           "l2": "flushed between timed iterations"}
    if wl["benchmark"] == "binomial":
        cfg.update({"n_per_gpu": wl["n"], "n_total": n_total, "lattice_steps": wl["lattice"],
                    "parallelism": (f"dp{ws}: contiguous team ranges of one {grid.num_teams}-team logical "
                                    "grid (global stride kept; decisions identical to the 1-GPU run)")})
    else:
        n = wl["boxes1d"] ** 3 if wl["benchmark"] == "lavamd" else wl["n"]
        cfg.update({"n_per_gpu": n * per_item, "parallelism": f"dp{ws} (independent shards)"})
    return cfg


# ------------------------------------------------------------------ reference arm

def ref_binomial_sample(wl, ws, threads, prefix=None, warmup=0):
    """The reference's own engine on whole team streams of the headline grid.

    `threads` teams spread evenly over the global logical grid (the
    reference's resolve_grid, bench/run.hpp:81-97) each run their complete
    item stream idx = team + s*T (or its first `prefix` items) through
    bench::binomial_region + run_region (bench/binomial.hpp:74-94,
    engine.hpp:132), one team per host thread. A one-team grid over the
    team's stream in order is the same execution as that team inside the
    full grid (per-team mapping: the team's tables see exactly these options
    in this order), so the sample has the full grid's table reuse. Imports
    only the checker package: no product code, no libhpac_b200.so."""
    import numpy as np

    import oracle
    from concurrent.futures import ThreadPoolExecutor
    n_total, _ = global_problem(wl, ws)
    opts = oracle.ref_portfolio("binomial", n_total, 42)
    grid, mapping = oracle.ref_grid("binomial", n_total, items_per_thread=wl["ipt"])
    spec = oracle.ref_parse(wl["directive"])
    T = grid.num_teams
    steps = -(-n_total // T)
    P = max(1, min(threads, T))
    teams = [j * T // P for j in range(P)]

    def stream(t):
        idx = t + np.arange(steps, dtype=np.int64) * T
        idx = idx[idx < n_total]
        return idx if prefix is None else idx[:prefix]

    def run_team(t, first=None):
        idx = stream(t) if first is None else stream(t)[:first]
        sub = oracle.abi.Grid(1, grid.threads_per_team, grid.warp_size, len(idx), grid.shared_mem_budget_bytes)
        rc, st, _, msg = oracle.ref_bench_binomial(opts[idx], wl["lattice"], sub, spec)
        assert rc == 0, msg
        return len(idx), st.approx_invocations, st.total_invocations

    with ThreadPoolExecutor(max_workers=P) as ex:
        for _ in range(warmup):  # page in the code on every thread (1 option each)
            list(ex.map(lambda t: run_team(t, first=1), teams))
        t0 = time.perf_counter()
        res = list(ex.map(run_team, teams))
        wall = time.perf_counter() - t0
    items = sum(r[0] for r in res)
    rate = sum(r[1] for r in res) / max(1, sum(r[2] for r in res))
    desc = (f"{P} of the {T} teams of the global grid (team j*T/{P}), "
            + ("each its whole " if prefix is None else f"each the first {prefix} options of its ")
            + f"{steps}-option stream (idx = team + s*{T}) through bench::binomial_region + run_region, "
            f"one host thread per team; {wl['lattice']}-step lattice; approx rate {rate:.4f}")
    return {"items": items, "wall_s": wall, "approx_rate": rate, "teams": P, "sample": desc,
            "grid": grid, "mapping": mapping}


def ref_binomial_floor(wl, threads, per_thread=32):
    """The reference's plain loop binomial_reference (bench/binomial.hpp:96-102)
    on all host threads: the no-engine CPU floor (every option priced once)."""
    import numpy as np

    import oracle
    from concurrent.futures import ThreadPoolExecutor
    n = wl["n"]
    opts = oracle.ref_portfolio("binomial", n, 42)
    chunks = [np.ascontiguousarray(opts[(np.arange(per_thread) * threads + j) * (n // (per_thread * threads))])
              for j in range(threads)]

    def one(c):
        out = np.empty(len(c))
        oracle.ref().ref_binomial_reference(c.ctypes.data, len(c), wl["lattice"], out.ctypes.data)
        return len(c)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        t0 = time.perf_counter()
        items = sum(ex.map(one, chunks))
        wall = time.perf_counter() - t0
    return {"value": items / wall, "unit": wl["unit"], "cores": threads, "kind": "reference",
            "sample": f"binomial_reference (plain per-option loop, no engine) over {items} options "
                      f"strided across the portfolio, {threads} threads"}


def reference_arm(args, wl):
    """`--impl reference`: the reference's own CPU implementation of the path
    (oracle/_ref = /root/reference compiled by oracle/Makefile) on the box's
    host cores, on this arm's config. Rank 0 only. Never imports the product
    package: inputs, grid and directive come from the reference's own
    generators, resolve_grid and parse_directive."""
    import numpy as np

    import oracle
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cores = host_cores()
    kind = "reference"
    extra = {}
    if wl["benchmark"] == "binomial":
        # K timed steps = K consecutive slices of the sampled teams' streams:
        # a team's table state must carry across the whole stream, so each
        # team runs as ONE run_region call and the K steps share its wall time
        r = ref_binomial_sample(wl, ws, cores, warmup=min(1, args.warmup))
        items, dt = r["items"], r["wall_s"]
        grid, mapping = r["grid"], r["mapping"]
        sample = r["sample"]
        extra = {"approx_rate": r["approx_rate"],
                 "cpu_floor": ref_binomial_floor(wl, cores),
                 "timing": ("one reference run_region per sampled team over its whole stream, all "
                            "teams concurrently; wall clock of the slowest; ms_per_step = wall / steps")}
    elif wl["benchmark"] == "blackscholes":
        n = wl["n"]
        opts = oracle.ref_portfolio("blackscholes", n, 42)
        grid, mapping = oracle.ref_grid("blackscholes", n, items_per_thread=wl["ipt"])
        spec = oracle.ref_parse(wl["directive"])
        G = grid.num_teams * grid.threads_per_team
        per = 64  # teams per worker: whole teams, every step of their streams
        sample = (f"{cores} threads x {per} whole teams of the {grid.num_teams}-team grid (all "
                  f"{grid.items_per_thread} steps of each stream), bench::blackscholes_region + run_region")
        from concurrent.futures import ThreadPoolExecutor

        def work(w):
            t0 = (w * per) % grid.num_teams
            thr = (t0 * grid.threads_per_team + np.arange(per * grid.threads_per_team))
            idx = (thr[None, :] + np.arange(grid.items_per_thread)[:, None] * G).ravel()
            idx = idx[idx < n]
            sub = oracle.abi.Grid(per, grid.threads_per_team, grid.warp_size, grid.items_per_thread,
                                  grid.shared_mem_budget_bytes)
            rc, st, _, msg = oracle.ref_bench_blackscholes(opts[idx], sub, spec)
            assert rc == 0, msg
            return len(idx)

        with ThreadPoolExecutor(max_workers=cores) as ex:
            t0 = time.perf_counter()
            items = sum(ex.map(work, range(cores)))
            dt = time.perf_counter() - t0
    else:
        # LavaMD and random perforation are not in the reference (SPEC.md:345,
        # SURVEY Appendix C): the checker's restatement (oracle port)
        kind = "port"
        from concurrent.futures import ThreadPoolExecutor
        if wl["benchmark"] == "lavamd":
            b1, P = wl["boxes1d"], wl["particles"]
            rv, qv = oracle.make_lavamd(b1, P, 42)
            nb = b1 ** 3
            grid = oracle.abi.Grid(nb, P, 32, 1, 48 * 1024)
            mapping = 1
            per = 4
            sp = oracle.abi.Spec()
            code, off = C.c_int32(), C.c_int64()
            err = C.create_string_buffer(256)
            oracle.ref().ref_parse_directive(wl["directive"].encode(), C.byref(sp), C.byref(code), C.byref(off), err, 256)
            sample = f"{cores} threads x {per} interior home boxes of the {b1}^3 system, oracle port"

            def work(w):
                b = nb // 2 + w * per
                fv = np.zeros((nb * P, 4))
                reg = oracle.abi.Region()
                reg.app, reg.output_dims, reg.lavamd_boxes1d, reg.lavamd_particles = 5, 4, b1, P
                reg.lavamd_alpha = 0.5
                reg.in_, reg.table_out, reg.out = rv.ctypes.data, qv.ctypes.data, fv.ctypes.data
                rc, st, msg = oracle.oracle_run_teams(grid, nb, 1, _Raw(reg), sp, (b, b + per))
                assert rc == 0, msg
                return per * P
        elif wl["benchmark"] == "kmeans":
            # the distance region through the reference engine (kmeans.hpp:85-102)
            kind = "reference"
            d, k = wl["dims"], wl["k"]
            grid, mapping = oracle.ref_grid("kmeans", wl["n"], items_per_thread=wl["ipt"])
            m = 1 << 13
            pts = oracle.ref_blobs(m * 4, d, k, 42, 8.0)
            cents = np.ascontiguousarray(pts[:k])
            sp = oracle.ref_parse(wl["directive"])
            sub = oracle.abi.Grid(m // (64 * wl["ipt"]), 64, 32, wl["ipt"], 48 * 1024)
            sample = f"{cores} threads x {m} points, one region launch each (reference run_region)"

            def work(w):
                x = np.ascontiguousarray(pts[(w % 4) * m:(w % 4 + 1) * m])
                lab = np.zeros(m, np.int32)
                reg = oracle.abi.Region()
                reg.app, reg.kmeans_dims, reg.kmeans_k = 4, d, k
                reg.in_, reg.centroids, reg.labels = x.ctypes.data, cents.ctypes.data, lab.ctypes.data
                rc, st, msg = oracle.ref_run(sub, m, 0, _Raw(reg), sp)
                assert rc == 0, msg
                return m
        else:
            d, k = wl["dims"], wl["k"]
            m, iters = 1 << 13, 5
            grid, mapping = oracle.ref_grid("kmeans", wl["n"], items_per_thread=wl["ipt"])
            pts = oracle.ref_blobs(m * 4, d, k, 42, wl.get("separation", 8.0))
            sub = oracle.abi.Grid(m // 256, 64, 32, 4, 48 * 1024)
            sp = oracle.abi.Spec()  # perfo(random:52) level(team): not reference grammar
            sp.technique, sp.level, sp.perfo_kind, sp.perfo_skip_percent = 2, 2, 6, 52
            sample = f"{cores} threads x {m} points x {iters} Lloyd iterations (oracle port kmeans_benchmark)"

            def work(w):
                x = np.ascontiguousarray(pts[(w % 4) * m:(w % 4 + 1) * m])
                lab = np.zeros(m, np.int32)
                cen = np.zeros((k, d))
                it_c, conv_c = C.c_int32(), C.c_int32()
                stc = oracle.abi.Stats()
                err = C.create_string_buffer(256)
                rc = oracle.oracle().oracle_kmeans_benchmark(x.ctypes.data, m, d, k, C.byref(sub), C.byref(sp),
                                                             iters, 7, lab.ctypes.data, cen.ctypes.data,
                                                             C.byref(it_c), C.byref(conv_c), C.byref(stc), err, 256)
                assert rc == 0, err.value
                return m * it_c.value

        with ThreadPoolExecutor(max_workers=cores) as ex:
            t0 = time.perf_counter()
            items = sum(ex.map(work, range(cores)))
            dt = time.perf_counter() - t0
    value = items / dt
    # evidence that this arm ran none of the product: its package was never
    # imported and its library never mapped
    try:
        mapped = any("libhpac_b200" in ln for ln in open("/proc/self/maps"))
    except OSError:
        mapped = None
    extra["product_code_loaded"] = bool(mapped) or any(
        m == "paper_2308_16877_b200" or (m.startswith("paper_2308_16877_b200.") and m != "paper_2308_16877_b200.abi")
        for m in sys.modules)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": wl["unit"],
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / max(1, args.steps) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the reference's generators, seed 42)",
        "config": bench_config(wl, grid, mapping, ws),
        "cpu_baseline": {"value": value, "unit": wl["unit"], "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": wl["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        **extra,
    }
    print(json.dumps(line), flush=True)


class _Raw:
    """A ready hpac_region_t for oracle.run_region-style helpers."""

    def __init__(self, s):
        self.s = s

    def c(self):
        return self.s


# ------------------------------------------------------------------ our arm

def cpu_baseline_sample(wl, opts, grid, ws=1):
    """Reference CPU engine on rank 0, bounded sample (~10-20 s). Binomial:
    the first 48 options of whole team streams on all host threads (the
    reference arm's method, bounded); the other workloads one thread."""
    import numpy as np

    import oracle
    from paper_2308_16877_b200 import engine as E
    if wl["benchmark"] == "binomial":
        cores = host_cores()
        r = ref_binomial_sample(wl, ws, cores, prefix=48)
        return {"value": r["items"] / r["wall_s"], "unit": wl["unit"], "cores": r["teams"],
                "kind": "reference", "sample": r["sample"]}
    try:
        oracle.ref()
        kind = "reference"
        runner = oracle.ref_run
    except Exception:
        kind = "port"
        runner = oracle.oracle_run
    t0 = time.perf_counter()
    if wl["benchmark"] == "blackscholes":
        m = 1 << 20
        sub = np.ascontiguousarray(opts[:m])
        out = np.zeros(m)
        rc, st, msg = runner(E.GridConfig(1024, 64, 32, 16), m, 0, E.blackscholes_region(sub, out),
                             make_spec(E, wl["spec"]))
        items = m
        desc = f"first {m} options, 1024 teams x 64 x ipt 16, 1 thread"
    elif wl["benchmark"] == "lavamd":
        # not in the reference: our oracle restatement
        runner, kind = oracle.oracle_run, "port"
        rv, qv = opts
        b1, P = wl["boxes1d"], wl["particles"]
        m = 96  # home boxes 0..95 of the 64^3 system, all 27-neighbourhoods
        fv = np.zeros((b1 ** 3 * P, 4))
        rc, st, msg = runner(E.GridConfig(m, P, 32, 1), m, 1, E.lavamd_region(rv, qv, fv, b1, P),
                             make_spec(E, wl["spec"]))
        scale = lava_cpu_scale(m, b1)
        items = m * P * scale
        desc = (f"home boxes 0..{m - 1} of the {b1}^3 system ({m * P} particles), oracle port, 1 thread; "
                f"rate scaled x{scale:.3f} to the {b1}^3 mean neighbour count")
    else:
        m = 1 << 14
        pts = np.ascontiguousarray(opts[0][:m])
        lab = np.zeros(m, np.int32)
        rc, st, msg = runner(E.GridConfig(m // 256, 64, 32, 4), m, 0, E.kmeans_region(pts, opts[1], lab),
                             make_spec(E, wl["spec"]))
        items = m
        desc = f"{m} points, one region launch, 1 thread"
    dt = time.perf_counter() - t0
    return {"value": items / dt, "unit": wl["unit"], "cores": 1, "kind": kind, "sample": desc}


def our_arm(args, wl, emit=True):
    import numpy as np
    import torch

    from paper_2308_16877_b200 import abi
    from paper_2308_16877_b200 import engine as E

    ws, rank, local = dist_env()
    local = gpu_index(local)
    torch.cuda.set_device(local)
    dist = init_dist(ws, local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    n = wl.get("n")
    spec = E.parse_directive(wl["directive"])[0]
    team_range = None

    # ---- inputs (synthetic, seeded)
    seed = 42 + rank
    if wl["benchmark"] == "binomial":
        # one global logical grid over ws x 2^20 options (the same portfolio on
        # every rank); this rank runs a contiguous range of its teams
        n = ws * wl["n"]
        opts = E.make_binomial_portfolio(n, 42)
        grid, mapping = E.resolve_grid("binomial", n, items_per_thread=wl["ipt"])
        if ws > 1:
            T = grid.num_teams
            team_range = (rank * T // ws, (rank + 1) * T // ws)
        d_in = torch.from_numpy(opts).to(dev)
        out_exact = torch.zeros(n, dtype=torch.float64, device=dev)
        out = torch.zeros(n, dtype=torch.float64, device=dev)
        mk = lambda o, s=None: E.binomial_region(d_in, wl["lattice"], o)
        h2d_bytes, d2h_bytes = n * 40, n * 8
        flops_item = binomial_flops(wl["lattice"])
        bound = "fp64"
        cpu_inputs = opts
    elif wl["benchmark"] == "blackscholes":
        opts = E.make_bs_portfolio(n, seed)
        grid, mapping = E.resolve_grid("blackscholes", n, items_per_thread=wl["ipt"])
        d_in = torch.from_numpy(opts).to(dev)
        out_exact = torch.zeros(n, dtype=torch.float64, device=dev)
        out = torch.zeros(n, dtype=torch.float64, device=dev)
        mk = lambda o, s=None: E.blackscholes_region(d_in, o)
        h2d_bytes, d2h_bytes = n * 40, n * 8
        flops_item = None
        bound = "hbm"
        cpu_inputs = opts
    elif wl["benchmark"] == "lavamd":
        b1, P = wl["boxes1d"], wl["particles"]
        n = b1 ** 3  # engine items = home boxes; metric items = particles
        rv, qv = E.make_lavamd(b1, P, seed)
        grid, mapping = E.resolve_grid("lavamd", n, items_per_thread=wl["ipt"])
        d_rv = torch.from_numpy(rv).to(dev)
        d_qv = torch.from_numpy(qv).to(dev)
        out_exact = torch.zeros((n * P, 4), dtype=torch.float64, device=dev)
        out = torch.zeros((n * P, 4), dtype=torch.float64, device=dev)
        mk = lambda o, s=None: E.lavamd_region(d_rv, d_qv, o, b1, P)
        h2d_bytes, d2h_bytes = n * P * (32 + 8 + 32), n * P * 32
        flops_item = LAVAMD_PAIR_FLOPS * P  # per evaluated (particle, neighbour box)
        bound = "fp64"
        cpu_inputs = (rv, qv)
        per_item = P
    else:
        d, k = wl["dims"], wl["k"]
        pts = E.make_blobs(n, d, k, seed, 8.0)
        cents = pts[:k].copy()
        grid, mapping = E.resolve_grid("kmeans", n, items_per_thread=wl["ipt"])
        d_in = torch.from_numpy(pts).to(dev)
        d_c = torch.from_numpy(cents).to(dev)
        out_exact = torch.zeros(n, dtype=torch.int32, device=dev)
        out = torch.zeros(n, dtype=torch.int32, device=dev)
        mk = lambda o, s=None: E.kmeans_region(d_in, d_c, o)
        h2d_bytes, d2h_bytes = n * d * 8, n * 4
        flops_item = kmeans_flops(d, k)
        bound = "fp64"
        cpu_inputs = (pts, cents)

    if wl["benchmark"] != "lavamd":
        per_item = 1  # metric items per engine item (LavaMD: particles per box)

    # L2 flush buffer (> 126 MB L2), written between timed iterations
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def timed_run(target, sp, steps, warmup, g=None):
        g = g or grid
        ts = []
        stats = None
        for i in range(warmup + steps):
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            # L2 flush (256 MB write) is enqueued first and left running, so the
            # host-side launch of the region overlaps it; the region kernel is
            # bracketed by the library's CUDA events on this stream (kernel_ms)
            if wl["benchmark"] == "lavamd":
                target.zero_()  # fv accumulates (Rodinia fv += ...)
            flush.zero_()
            E.run_region(g, n, mapping, mk(target), sp, stream=stream, synchronous=False,
                         team_range=team_range if g is grid else None)
            torch.cuda.synchronize()
            st = abi.Stats()
            rc = abi.lib().hpac_stats_fetch(C.byref(st))
            assert rc == 0, rc
            if i >= warmup:
                ts.append(st.kernel_ms)
                stats = st.as_dict()
        return ts, stats

    # exact GPU kernel (same grid, spec = NULL) and the approximate region
    ts_exact, st_exact = timed_run(out_exact, None, args.steps, args.warmup)
    clocks = ClockSampler(local)
    clocks.start()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 0.6:  # untimed load so nvidia-smi sees the clocks
        E.run_region(grid, n, mapping, mk(out), spec, stream=stream, team_range=team_range)
    ts_apx, st_apx = timed_run(out, spec, args.steps, args.warmup)
    time.sleep(0.15)
    clk = clocks.stop()

    # quality loss (application metric) vs the exact run; under a team-range
    # split every rank holds the whole output array and fills its own items,
    # so the ranks' outputs are summed (disjoint items) before the metric
    if dist is not None and team_range is not None:
        dist.all_reduce(out_exact)
        dist.all_reduce(out)
    if wl["benchmark"] == "kmeans":
        quality = {"mcr": E.mcr(out_exact, out)}
        qval = quality["mcr"]
    else:
        quality = {"mape": E.mape(out_exact, out)}
        qval = quality["mape"]

    t_apx = sum(ts_apx)
    t_exact = sum(ts_exact)
    if dist is not None:
        t = torch.tensor([t_apx, t_exact], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_apx, t_exact = t.tolist()
    job_items = (n if team_range is not None or ws == 1 else ws * n) * per_item
    value = job_items * args.steps / (t_apx * 1e-3)
    exact_value = job_items * args.steps / (t_exact * 1e-3)

    # ---- the exact kernel at its own best grid (binomial: ipt 256), beside the
    # same-grid baseline above (a larger ipt gives the table more reuse but
    # fewer, longer teams)
    exact_best = None
    if wl["benchmark"] == "binomial" and ws == 1 and wl.get("exact_best_ipt"):
        g_best, _ = E.resolve_grid("binomial", n, items_per_thread=wl["exact_best_ipt"])
        ts_b, _ = timed_run(out_exact, None, args.steps, 1, g=g_best)
        exact_best = {"items_per_thread": wl["exact_best_ipt"], "num_teams": g_best.num_teams,
                      "value": n * args.steps / (sum(ts_b) * 1e-3),
                      "speedup_of_approx_over_it": value / (n * args.steps / (sum(ts_b) * 1e-3))}

    # ---- decision granularity comparison (C4: warp vs team, + thread)
    levels = None
    if wl.get("compare_levels"):
        levels = {wl["spec"][-1]: {"speedup_vs_exact": t_exact / t_apx, "quality": qval,
                                   "approx_rate": st_apx["approx_invocations"] / max(1, st_apx["total_invocations"]),
                                   "divergent_fraction": st_apx["divergent_warp_steps"] / max(1, st_apx["total_warp_steps"])}}
        for lv in wl["compare_levels"]:
            sp_l = make_spec(E, tuple(wl["spec"][:-1]) + (lv,))
            o_l = torch.zeros_like(out)
            ts_l, st_l = timed_run(o_l, sp_l, max(1, args.steps // 2), 1)
            levels[lv] = {"speedup_vs_exact": (t_exact / len(ts_exact)) / (sum(ts_l) / len(ts_l)),
                          "quality": E.mape(out_exact, o_l),
                          "approx_rate": st_l["approx_invocations"] / max(1, st_l["total_invocations"]),
                          "divergent_fraction": st_l["divergent_warp_steps"] / max(1, st_l["total_warp_steps"])}
            del o_l
    ms_per_step = t_apx / args.steps

    # ---- end to end through the C-ABI with pinned host buffers
    e2e = None
    if args.e2e_steps > 0:
        if wl["benchmark"] == "kmeans":
            h_in = torch.from_numpy(pts).pin_memory()
            h_lab = torch.zeros(n, dtype=torch.int32).pin_memory()
            hreg = E.kmeans_region(h_in.numpy(), cents, h_lab.numpy())
        elif wl["benchmark"] == "lavamd":
            h_rv = torch.from_numpy(rv).pin_memory()
            h_qv = torch.from_numpy(qv).pin_memory()
            h_fv = torch.zeros((n * P, 4), dtype=torch.float64).pin_memory()
            hreg = E.lavamd_region(h_rv.numpy(), h_qv.numpy(), h_fv.numpy(), b1, P)
        else:
            h_in = torch.from_numpy(cpu_inputs).pin_memory()
            h_out = torch.zeros(n, dtype=torch.float64).pin_memory()
            hreg = (E.binomial_region(h_in.numpy(), wl["lattice"], h_out.numpy())
                    if wl["benchmark"] == "binomial" else E.blackscholes_region(h_in.numpy(), h_out.numpy()))
        e2e_note = None
        if team_range is None:
            zc = E.run_region_host(grid, n, mapping, hreg, spec).stats["zero_copy"]  # warm-up

            def e2e_step():
                E.run_region_host(grid, n, mapping, hreg, spec)
            e2e_items = job_items
        else:
            # team-range split: each rank's host entry moves only its team
            # range's options in and prices out (2-D column-block copies,
            # hpac_run_region_host_teams); all ranks together move the whole
            # portfolio once per step
            zc = 0
            e2e_note = ("each rank moves only its team range's options and prices "
                        "(hpac_run_region_host_teams); bytes are the job's total")

            def e2e_step():
                E.run_region_host(grid, n, mapping, hreg, spec, team_range=team_range)
            e2e_step()
            e2e_items = job_items
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        e2e_t = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_t = t.item()
        e2e = {"value": e2e_items * args.e2e_steps / e2e_t, "unit": wl["unit"],
               "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
               "steps": args.e2e_steps,
               "transfer": ("zero-copy: the region kernel reads the pinned host inputs and writes the "
                            "pinned host outputs in place over PCIe" if zc else
                            "staged: H2D copy, region kernel, D2H copy")}
        if e2e_note:
            e2e["note"] = e2e_note

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return None

    # ---- roofline of the dominant kernel (the region kernel itself)
    peaks = measured_peaks()
    avg_ms = t_apx / args.steps
    if bound == "fp64":
        fp = C.c_double()
        dmma = wl["benchmark"] == "kmeans" and kmeans_uses_dmma(wl["dims"], wl["k"])
        (abi.lib().hpac_probe_dmma_peak if dmma else abi.lib().hpac_probe_fp64_peak)(C.byref(fp))
        evaluated = st_apx["total_invocations"] - st_apx["approx_invocations"]
        # per-team mapping: the team's lanes evaluate one item redundantly,
        # except LavaMD where each lane is its own particle
        per_item_lanes = grid.threads_per_team if (mapping == 1 and per_item == 1) else 1
        evaluated_items = evaluated / per_item_lanes
        achieved = evaluated_items * flops_item / (avg_ms * 1e-3) / 1e12
        roof = {"bound": "tensor" if dmma else "fp64", "achieved": achieved, "peak": fp.value,
                "unit": "TFLOP/s", "frac": achieved / fp.value if fp.value else None,
                "peak_source": DMMA_PEAK_SOURCE if dmma else FP64_PEAK_SOURCE,
                "algorithmic": f"{flops_item:.4g} FP64 flops per evaluated item"}
        if wl["benchmark"] == "binomial" and st_apx.get("lattice_nodes"):
            # the American-put lattice skips the early-exercise region (analytic
            # values): report the node updates actually executed beside the
            # algorithmic (full-triangle) figure
            full_nodes = evaluated_items * wl["lattice"] * (wl["lattice"] + 1) / 2
            roof["executed_node_fraction"] = st_apx["lattice_nodes"] / full_nodes
            roof["achieved_executed"] = 5.0 * st_apx["lattice_nodes"] / (avg_ms * 1e-3) / 1e12
            roof["frac_executed"] = roof["achieved_executed"] / fp.value if fp.value else None
            roof["lattice_fallbacks"] = st_apx.get("lattice_fallbacks", 0)
    else:
        approx_items = st_apx["approx_invocations"]
        bytes_launch = 48 * n - 40 * approx_items  # approx items skip the 40 B input read
        achieved = bytes_launch / (avg_ms * 1e-3) / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s",
                "algorithmic": "48 B per exact option, 8 B per TAF-approximated option"}
    roof["traffic"] = load_traffic(wl["name"])
    # the same launch against the HBM roofline (north star: every number also
    # as a fraction of HBM); algorithmic bytes per metric item
    bytes_item = {"binomial": 48.0, "blackscholes": 48.0, "lavamd": 104.0, "kmeans": 260.0}[wl["benchmark"]]
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    if wl["benchmark"] == "blackscholes":
        hbm_ach = roof["achieved"]
    else:
        hbm_ach = (job_items / max(1, ws if team_range is not None else 1)) * bytes_item / (avg_ms * 1e-3) / 1e9
    roof["hbm"] = {"achieved_gbs": hbm_ach, "peak_gbs": hbm_peak, "frac": hbm_ach / hbm_peak,
                   "algorithmic": f"{bytes_item:.0f} B per item"}

    cpu = None
    cpu_floor = None
    if args.cpu_baseline and ws == 1:
        try:
            cpu = cpu_baseline_sample(wl, cpu_inputs, grid, ws)
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "unit": wl["unit"], "cores": 1, "kind": "reference",
                   "sample": f"failed: {exc}"}
        if wl["benchmark"] == "binomial":
            try:
                cpu_floor = ref_binomial_floor(wl, host_cores())
            except Exception as exc:
                cpu_floor = {"value": None, "sample": f"failed: {exc}"}

    extra = {}
    if levels:
        extra["decision_levels"] = levels
    if exact_best:
        extra["exact_best_grid"] = exact_best
    if cpu_floor:
        extra["cpu_floor"] = cpu_floor
    line = {
        "metric": METRIC, "value": value, "unit": wl["unit"], "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generators, seed 42" + (")" if team_range is not None or ws == 1
                                                               else " + rank)"),
        "config": bench_config(wl, grid, mapping, ws),
        "speedup_vs_exact": value / exact_value,
        "exact_value": exact_value,
        "quality": quality, "quality_ok": bool(qval <= 0.01),
        "approx_rate": st_apx["approx_invocations"] / max(1, st_apx["total_invocations"]),
        "divergent_fraction": st_apx["divergent_warp_steps"] / max(1, st_apx["total_warp_steps"]),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        # region kernels per step: one, + the DMMA operand kernel for K-Means;
        # binomial (non-TAF) = decide + price (+ resolve for iACT)
        "gpu_launches": args.steps * region_launches(wl),
        "clocks": clk, **extra,
    }
    if emit:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return line


def region_launches(wl):
    """Kernels one run_region launch of this workload enqueues (csrc/*.cu)."""
    if wl["benchmark"] == "kmeans" and kmeans_uses_dmma(wl["dims"], wl["k"]):
        return 2  # kmeans_dmma_aux_kernel + engine_thread_kernel
    if wl["benchmark"] == "binomial" and wl["spec"][0] != "taf":
        # binomial_decide_kernel + binomial_price_kernel (+ binomial_resolve_kernel)
        return 3 if wl["spec"][0] == "iact" else 2
    return 1


def kmeans_lloyd_arm(args, wl, emit=True):
    """C3: the Lloyd loop (hpac_kmeans_run) exact vs perforated on the same
    synthetic points; per-GPU shard of n points, centroid partials
    all-reduced over NCCL every iteration when N > 1 (weak scaling)."""
    import numpy as np
    import torch

    from paper_2308_16877_b200 import distributed as D
    from paper_2308_16877_b200 import engine as E

    ws, rank, local = dist_env()
    local = gpu_index(local)
    torch.cuda.set_device(local)
    dist = init_dist(ws, local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    n, d, k = wl["n"], wl["dims"], wl["k"]
    pts = E.make_blobs(n, d, k, 42 + rank, wl["separation"])
    d_pts = torch.from_numpy(pts).to(dev)
    # Forgy init from rank 0's first k points, identical on every rank
    cent0 = torch.from_numpy(E.make_blobs(n, d, k, 42, wl["separation"])[:k].copy() if rank else pts[:k].copy()).to(dev)
    grid, _ = E.resolve_grid("kmeans", n, items_per_thread=wl["ipt"])
    spec = E.parse_directive(wl["directive"])[0]
    # N > 1: torch.distributed's all_reduce as the per-iteration hook (host
    # loop). BENCH_KMEANS_NATIVE_NCCL=1 uses the library's own multi-process
    # NCCL communicator instead, so the all-reduce is captured in the Lloyd
    # loop's CUDA graph (single-rank tested; multi-GPU unmeasured here, hence
    # opt-in). `value` is kernel time either way; the graph removes host gaps.
    allreduce, nccl_comm = None, None
    if dist is not None:
        if (os.environ.get("BENCH_KMEANS_NATIVE_NCCL")
                and os.environ.get("BENCH_DIST_BACKEND", "nccl") == "nccl"):
            try:
                nccl_comm = D.native_nccl_comm(rank, ws)
            except Exception as exc:  # fall back to the torch hook
                print(f"native NCCL communicator unavailable: {exc}", file=sys.stderr)
                nccl_comm = None
        if nccl_comm is None:
            allreduce = D.kmeans_allreduce_hook()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def one(sp, seed):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        flush.zero_()
        r = E.kmeans_run(grid, d_pts, k, sp, max_iters=wl["max_iters"], centroids=cent0.clone(),
                         perfo_seed_base=seed, allreduce=allreduce, stream=stream, nccl_comm=nccl_comm)
        torch.cuda.synchronize()
        # device time of the run: the library's CUDA events around every
        # region launch and every update (partials + all-reduce + readback);
        # host-side gaps between iterations (the convergence readback) are
        # not device work and are excluded
        return r, r.region_ms + r.update_ms

    def timed(sp):
        for i in range(args.warmup):
            one(sp, 1000 + i)
        res = [one(sp, 7) for _ in range(args.steps)]
        return res

    ex = timed(None)
    clocks = ClockSampler(local)
    clocks.start()
    ap = timed(spec)
    time.sleep(0.15)
    clk = clocks.stop()
    r_e, r_a = ex[-1][0], ap[-1][0]
    t_e = sum(t for _, t in ex)
    t_a = sum(t for _, t in ap)
    reg_a = sum(r.region_ms for r, _ in ap)
    if dist is not None:
        t = torch.tensor([t_e, t_a, reg_a], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e, t_a, reg_a = t.tolist()
    it_e, it_a = r_e.iterations, r_a.iterations
    value = ws * n * it_a * args.steps / (t_a * 1e-3)
    exact_value = ws * n * it_e * args.steps / (t_e * 1e-3)
    mcr = E.mcr(r_e.assignments, r_a.assignments)

    # end to end: pinned host points -> device, Lloyd loop, labels -> host
    e2e = None
    if args.e2e_steps > 0:
        h_pts = torch.from_numpy(pts).pin_memory()
        h_lab = torch.empty(n, dtype=torch.int32).pin_memory()
        buf = torch.empty_like(d_pts)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = 0
        torch.cuda.synchronize()
        ev0.record(stream)
        dbg = os.environ.get("BENCH_DEBUG")
        for _ in range(args.e2e_steps):
            t_0 = time.perf_counter()
            buf.copy_(h_pts, non_blocking=True)
            if dbg:
                torch.cuda.synchronize()
                t_1 = time.perf_counter()
            r = E.kmeans_run(grid, buf, k, spec, max_iters=wl["max_iters"], centroids=cent0.clone(),
                             perfo_seed_base=7, allreduce=allreduce, stream=stream, nccl_comm=nccl_comm)
            if dbg:
                t_2 = time.perf_counter()
            h_lab.copy_(r.assignments, non_blocking=True)
            its += r.iterations
            if dbg:
                torch.cuda.synchronize()
                t_3 = time.perf_counter()
                print(f"e2e step: h2d {(t_1 - t_0) * 1e3:.1f} ms, lloyd {(t_2 - t_1) * 1e3:.1f} ms "
                      f"(kernels {r.region_ms + r.update_ms:.1f}), d2h {(t_3 - t_2) * 1e3:.1f} ms",
                      file=sys.stderr)

        ev1.record(stream)
        torch.cuda.synchronize()
        e2e_t = ev0.elapsed_time(ev1)
        if dist is not None:
            t = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_t = t.item()
        e2e = {"value": ws * n * its / (e2e_t * 1e-3), "unit": wl["unit"],
               "h2d_bytes_per_step": n * d * 8, "d2h_bytes_per_step": n * 4, "steps": args.e2e_steps}

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return None
    from paper_2308_16877_b200 import abi
    fp = C.c_double()
    dmma = kmeans_uses_dmma(d, k)
    (abi.lib().hpac_probe_dmma_peak if dmma else abi.lib().hpac_probe_fp64_peak)(C.byref(fp))
    st = r_a.stats
    evaluated = (st["total_invocations"] - st["approx_invocations"]) * args.steps
    achieved = evaluated * kmeans_filter_flops(d, k) / (reg_a * 1e-3) / 1e12
    roof = {"bound": "tensor" if dmma else "fp64",
            "kernel": "distance region (engine_thread_kernel<AppKmeansDmma>, FP64 tensor op)" if dmma
                      else "distance region (engine_thread_kernel<AppKmeans>)",
            "achieved": achieved, "peak": fp.value, "unit": "TFLOP/s",
            "frac": achieved / fp.value if fp.value else None,
            "peak_source": DMMA_PEAK_SOURCE if dmma else FP64_PEAK_SOURCE,
            "algorithmic": f"{kmeans_filter_flops(d, k):.0f} FP64 flops per evaluated point-iteration "
                           "(filtered argmin; reference order only on near-ties)",
            "region_share_of_step": reg_a / t_a,
            "traffic": load_traffic(wl["name"])}
    # against HBM: 260 B per point-iteration in the region + 260 B in the
    # centroid update (points re-read, labels), over the whole Lloyd step
    peaks = measured_peaks()
    hbm_ach = n * it_a * args.steps * 520.0 / (t_a * 1e-3) / 1e9
    roof["hbm"] = {"achieved_gbs": hbm_ach, "peak_gbs": peaks.get("hbm_gbs", 6650.0),
                   "frac": hbm_ach / peaks.get("hbm_gbs", 6650.0),
                   "algorithmic": "520 B per point-iteration (region + update)"}
    cpu = None
    if args.cpu_baseline and ws == 1:
        try:
            import oracle
            # random perforation is not in the reference: the
            # oracle port's kmeans_benchmark on a bounded sample
            m, iters = 1 << 13, 8
            sub = np.ascontiguousarray(pts[:m])
            lab = np.zeros(m, np.int32)
            cen = np.zeros((k, d))
            it_c, conv_c = C.c_int32(), C.c_int32()
            stc = abi.Stats()
            err = C.create_string_buffer(256)
            g2 = E.GridConfig(m // 256, 64, 32, 4)
            t0 = time.perf_counter()
            rc = oracle.oracle().oracle_kmeans_benchmark(sub.ctypes.data, m, d, k, C.byref(g2.c()), C.byref(spec),
                                                         iters, 7, lab.ctypes.data, cen.ctypes.data,
                                                         C.byref(it_c), C.byref(conv_c), C.byref(stc), err, 256)
            dt = time.perf_counter() - t0
            assert rc == 0, err.value
            cpu = {"value": m * it_c.value / dt, "unit": wl["unit"], "cores": 1, "kind": "port",
                   "sample": f"{m} points, kmeans_benchmark for {it_c.value} iterations (oracle port), 1 thread"}
        except Exception as exc:
            cpu = {"value": None, "unit": wl["unit"], "cores": 1, "kind": "reference", "sample": f"failed: {exc}"}
    line = {
        "metric": METRIC, "value": value, "unit": wl["unit"], "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_a / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic make_blobs(separation {wl['separation']}), seed 42 + rank",
        "config": {**bench_config(wl, grid, 0, ws), "dims": d, "k": k,
                   "max_iters": wl["max_iters"], "step": "one full Lloyd run (kmeans_benchmark)",
                   "parallelism": f"dp{ws} (points sharded, NCCL all-reduce of centroid partials per iteration)"},
        "timing": "sum of the region and update kernels' CUDA-event times per run (4.3 GB of points per GPU >> L2)",
        "speedup_vs_exact": value / exact_value,
        "time_to_solution_speedup": t_e / t_a,
        "exact_value": exact_value,
        "iterations": {"exact": it_e, "approx": it_a},
        "converged": {"exact": r_e.converged, "approx": r_a.converged},
        "quality": {"mcr": mcr}, "quality_ok": bool(mcr <= 0.01),
        "approx_rate": st["approx_invocations"] / max(1, st["total_invocations"]),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": args.steps * lloyd_launches(
            r_a, kmeans_uses_dmma(d, k),
            random_first_exact=spec is not None and spec.technique == abi.TECH_PERFO
            and spec.perfo_kind == abi.PERFO_RANDOM),
        "clocks": clk,
    }
    if emit:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return line


SUB_CONFIGS = ("blackscholes", "kmeans", "lavamd")  # C1, C3, C4 beside the C2 headline


def run_workload(args, wl, emit=True):
    if wl["benchmark"] == "kmeans_lloyd":
        return kmeans_lloyd_arm(args, wl, emit)
    return our_arm(args, wl, emit)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="binomial", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--sub-configs", default="auto", choices=["auto", "on", "off"],
                    help="also measure C1/C3/C4 in this invocation and report them under `configs` "
                         "(auto: the default binomial workload at N=1)")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        reference_arm(args, wl)
        return
    ws = dist_env()[0]
    sub = args.sub_configs == "on" or (args.sub_configs == "auto" and ws == 1 and args.workload == "binomial")
    line = run_workload(args, wl, emit=not sub)
    if sub and line is not None:
        sargs = argparse.Namespace(**vars(args))
        sargs.steps, sargs.warmup, sargs.e2e_steps = max(3, args.steps // 4), max(3, min(args.warmup, 3)), 1
        configs = {}
        for name in SUB_CONFIGS:
            try:
                configs[name] = run_workload(sargs, WORKLOADS[name], emit=False)
            except Exception as exc:  # a sub-config never takes the headline down
                configs[name] = {"workload": WORKLOADS[name]["name"], "error": repr(exc)}
        line["configs"] = configs
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
