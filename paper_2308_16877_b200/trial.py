"""Trial records and the trial runner over the C-ABI.

Mirrors the reference's TrialRecord CSV (trial.hpp:16-54, header
kTrialCsvHeader) and run_trial (bench/run.hpp:172-232): one sweep point =
one directive on one application workload; the accurate baseline runs on the
same logical grid; the record carries the application's error metric (MAPE,
or MCR for K-Means), the approximation rate and the divergent warp-step
fraction. The reference's cost-model columns hold MEASURED device time here:
baseline_cost / approx_cost are milliseconds of the region kernel(s) (the
whole Lloyd loop for K-Means) and est_speedup is the items/s ratio (per
Lloyd iteration for K-Means). Three columns are appended: items_per_s,
time_to_solution_speedup and workload (the generator/shape parameters the
reference keeps in BenchmarkParams, e.g. K-Means separation).

Apps run on the current CUDA device; a FAILED record (status/reason) is
written for configurations the engine rejects (run.hpp:224-230).
"""
from __future__ import annotations

import csv
import io
import math
from dataclasses import dataclass, field, fields

REF_HEADER = ("benchmark,technique,directive,level,num_teams,threads_per_team,warp_size,"
              "items_per_thread,n,seed,trial,status,reason,error_metric,error_value,approx_rate,"
              "divergent_fraction,baseline_cost,approx_cost,est_speedup,baseline_iters,approx_iters")
EXTRA = ("items_per_s", "time_to_solution_speedup", "workload")
HEADER = REF_HEADER + "," + ",".join(EXTRA)

# region array sections per app (the directive grammar needs in/out clauses,
# docs/directives.md); the engine only validates them
SECTIONS = {
    "blackscholes": "in(opt[i:5]) out(price[i])",
    "binomial": "in(opt[i:5]) out(price[i])",
    "kmeans": "in(pt[i:32]) out(dist[i:64])",
    "lavamd": "out(fv[i:4])",
}


@dataclass
class TrialRecord:
    benchmark: str
    technique: str
    directive: str
    level: str = "thread"
    num_teams: int = 0
    threads_per_team: int = 0
    warp_size: int = 0
    items_per_thread: int = 0
    n: int = 0
    seed: int = 0
    trial: int = 0
    status: str = "OK"
    reason: str = ""
    error_metric: str = ""
    error_value: float = 0.0
    approx_rate: float = 0.0
    divergent_fraction: float = 0.0
    baseline_cost: float = 0.0
    approx_cost: float = 0.0
    est_speedup: float = 0.0
    baseline_iters: int = 0
    approx_iters: int = 0
    items_per_s: float = 0.0
    time_to_solution_speedup: float = 0.0
    workload: str = ""  # generator / shape parameters the reference keeps in BenchmarkParams

    def sort_key(self):
        """trial.hpp:40-47: every configuration field, canonical order."""
        return "\x1f".join(str(x) for x in (self.benchmark, self.technique, self.directive, self.level,
                                            self.num_teams, self.threads_per_team, self.warp_size,
                                            self.items_per_thread, self.n, self.seed, self.trial,
                                            self.workload))


def fmt_num(v):
    """Shortest round-trip doubles (fmtnum.hpp:13-19); ints as ints."""
    if isinstance(v, bool):
        return str(int(v))
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        if math.isnan(v):
            return "nan"
        if math.isinf(v):
            return "inf" if v > 0 else "-inf"
        return repr(v)
    return str(v)


def to_csv_row(rec: TrialRecord) -> str:
    out = io.StringIO()
    csv.writer(out, lineterminator="").writerow([fmt_num(getattr(rec, f.name)) for f in fields(rec)])
    return out.getvalue()


def from_csv_row(line: str) -> TrialRecord:
    vals = next(csv.reader([line]))
    kw = {}
    for f, v in zip(fields(TrialRecord), vals):
        if f.type in ("int", int):
            kw[f.name] = int(v)
        elif f.type in ("float", float):
            kw[f.name] = float(v)
        else:
            kw[f.name] = v
    return TrialRecord(**kw)


def technique_name(spec) -> str:
    from . import abi
    if spec is None:
        return "none"
    return {abi.TECH_TAF: "taf", abi.TECH_IACT: "iact", abi.TECH_PERFO: "perfo"}[spec.technique]


def level_name(spec) -> str:
    if spec is None:
        return "thread"
    return {0: "thread", 1: "warp", 2: "team"}[spec.level]


@dataclass
class Workload:
    """Application inputs resident on the device, plus cached baselines."""
    app: str
    n: int
    ipt: int
    extra: dict = field(default_factory=dict)
    _cache: dict = field(default_factory=dict)


def make_workload(app: str, n: int, ipt: int, seed: int = 42, **extra) -> Workload:
    import torch
    from . import engine as E
    w = Workload(app, n, ipt, dict(extra))
    w.extra["seed"] = seed
    if app == "blackscholes":
        w.extra["inputs"] = torch.from_numpy(E.make_bs_portfolio(n, seed)).cuda()
    elif app == "binomial":
        w.extra["inputs"] = torch.from_numpy(E.make_binomial_portfolio(n, seed)).cuda()
        w.extra.setdefault("lattice", 1024)
    elif app == "kmeans":
        d, k = extra.get("dims", 32), extra.get("k", 64)
        pts = E.make_blobs(n, d, k, seed, extra.get("separation", 30.0))
        w.extra.update(dims=d, k=k, points=torch.from_numpy(pts).cuda(),
                       cent0=torch.from_numpy(pts[:k].copy()).cuda())
        w.extra.setdefault("max_iters", 40)
    elif app == "lavamd":
        b1, P = extra.get("boxes1d", 32), extra.get("particles", 128)
        rv, qv = E.make_lavamd(b1, P, seed)
        w.n = b1 ** 3
        w.extra.update(boxes1d=b1, particles=P, rv=torch.from_numpy(rv).cuda(), qv=torch.from_numpy(qv).cuda())
    else:
        raise ValueError(f"unknown app {app}")
    return w


def _grid(w: Workload):
    from . import engine as E
    return E.resolve_grid(w.app, w.n, items_per_thread=w.ipt)


def _run_once(w: Workload, spec, seed_base=7):
    """One timed run: (ms, items, out tensor, stats, iterations)."""
    import torch
    from . import engine as E
    grid, mp = _grid(w)
    if w.app == "kmeans":
        r = E.kmeans_run(grid, w.extra["points"], w.extra["k"], spec, max_iters=w.extra["max_iters"],
                         centroids=w.extra["cent0"].clone(), perfo_seed_base=seed_base)
        return r.region_ms + r.update_ms, w.n * r.iterations, r.assignments, r.stats, r.iterations
    if w.app == "lavamd":
        P = w.extra["particles"]
        out = torch.zeros((w.n * P, 4), dtype=torch.float64, device="cuda")
        lr = E.run_region(grid, w.n, mp, E.lavamd_region(w.extra["rv"], w.extra["qv"], out, w.extra["boxes1d"], P),
                          spec)
        return lr.kernel_ms, w.n * P, out, lr.stats, 0
    out = torch.zeros(w.n, dtype=torch.float64, device="cuda")
    if w.app == "blackscholes":
        reg = E.blackscholes_region(w.extra["inputs"], out)
    else:
        reg = E.binomial_region(w.extra["inputs"], w.extra["lattice"], out)
    lr = E.run_region(grid, w.n, mp, reg, spec)
    return lr.kernel_ms, w.n, out, lr.stats, 0


def run_trial(w: Workload, directive: str, trial: int = 0, reps: int = 2) -> TrialRecord:
    """bench::run_trial (bench/run.hpp:172-232) on the device."""
    from . import engine as E
    grid, _ = _grid(w)
    params = {k: v for k, v in w.extra.items() if isinstance(v, (int, float, str)) and k != "seed"}
    rec = TrialRecord(benchmark=w.app, technique="none", directive=directive, n=w.n,
                      workload=";".join(f"{k}={v}" for k, v in sorted(params.items())),
                      num_teams=grid.num_teams, threads_per_team=grid.threads_per_team,
                      warp_size=grid.warp_size, items_per_thread=grid.items_per_thread,
                      seed=w.extra["seed"], trial=trial,
                      error_metric="mcr" if w.app == "kmeans" else "mape")
    try:
        spec, canon = E.parse_directive(directive)
        rec.directive, rec.technique, rec.level = canon, technique_name(spec), level_name(spec)
        if "base" not in w._cache:  # BaselineCache (run.hpp:109-121)
            _run_once(w, None)  # warm-up
            w._cache["base"] = min((_run_once(w, None) for _ in range(reps)), key=lambda t: t[0])
        b_ms, b_items, b_out, _, b_it = w._cache["base"]
        _run_once(w, spec)
        a_ms, a_items, a_out, st, a_it = min((_run_once(w, spec) for _ in range(reps)), key=lambda t: t[0])
    except (E.ConfigError, E.ArenaOverflowError, E.BarrierDivergenceError, E.UnsupportedError,
            E.DirectiveError) as exc:
        rec.status, rec.reason = "FAILED", f"{type(exc).__name__}: {exc}"
        return rec
    rec.error_value = E.mcr(b_out, a_out) if w.app == "kmeans" else E.mape(b_out, a_out)
    rec.approx_rate = st["approx_invocations"] / max(1, st["total_invocations"])
    rec.divergent_fraction = st["divergent_warp_steps"] / max(1, st["total_warp_steps"])
    rec.baseline_cost, rec.approx_cost = b_ms, a_ms
    rec.baseline_iters, rec.approx_iters = b_it, a_it
    rec.items_per_s = a_items / (a_ms * 1e-3)
    b_rate = b_items / (b_ms * 1e-3)
    rec.est_speedup = rec.items_per_s / b_rate  # throughput ratio (per iteration for K-Means)
    rec.time_to_solution_speedup = b_ms / a_ms
    return rec
