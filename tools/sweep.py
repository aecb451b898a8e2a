#!/usr/bin/env python3
"""C5: approximation-parameter sweep across the four applications.

The reference's execute_sweep (harness/sweep.hpp:203-289) on the C-ABI:
Cartesian points (technique x parameters x level) per application, one
TrialRecord CSV row each (paper_2308_16877_b200/trial.py), streamed to a
resumable `<out>.part` file, then a canonical sorted rewrite and an atomic
rename (sweep.hpp:195-289) plus a JSON sidecar.

One GPU: python tools/sweep.py --out sweep.csv [--apps blackscholes,binomial,kmeans,lavamd] [--quick]
N GPUs:  torchrun --nproc-per-node N tools/sweep.py --out sweep.csv
         (point i runs on rank i mod N — one sweep point per GPU at a time,
          like --jobs; every rank streams to its own <out>.part.<rank>; rank 0
          merges once all ranks are done)
A killed sweep resumes: points already in the .part files are not re-run.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2308_16877_b200 import trial as T  # noqa: E402


def points(apps, quick=False):
    """Deterministic point list: (app, workload kwargs, directive)."""
    out = []
    S = T.SECTIONS
    if "blackscholes" in apps:
        wl = dict(n=1 << 22, ipt=16)
        for lv in ("thread", "warp"):
            for h, p in ((2, 1), (5, 1), (5, 2), (5, 8)):
                for thr in ((0.5,) if quick else (0.1, 0.5, 1.0)):
                    out.append(("blackscholes", wl, f"memo(out:{h}:{p}:{thr}) {S['blackscholes']} level({lv})"))
        for ts, thr in ((2, 0.5), (4, 0.3), (8, 0.3)):
            for lv in ("thread", "warp"):
                out.append(("blackscholes", wl, f"memo(in:{ts}:{thr}) {S['blackscholes']} level({lv})"))
        for kind, arg in (("small", 2), ("small", 4), ("large", 2), ("random", 10), ("random", 25)):
            out.append(("blackscholes", wl, f"perfo({kind}:{arg}) {S['blackscholes']}"))
    if "binomial" in apps:
        for ipt in ((128,) if quick else (64, 128, 384)):
            wl = dict(n=1 << 18, ipt=ipt)
            for ts in (2, 4, 8):
                for thr in ((0.5,) if quick else (0.25, 0.4, 0.5, 1.0)):
                    out.append(("binomial", wl, f"memo(in:{ts}:{thr}) {S['binomial']} level(team)"))
            for kind, arg in (("small", 4), ("random", 25)):
                out.append(("binomial", wl, f"perfo({kind}:{arg}) {S['binomial']} level(team)"))
    if "kmeans" in apps:
        for sep in ((30.0,) if quick else (8.0, 30.0)):
            wl = dict(n=1 << 22, ipt=4, separation=sep)
            for p in (10, 25, 50):
                for lv in ("thread", "warp"):
                    out.append(("kmeans", wl, f"perfo(random:{p}) {S['kmeans']} level({lv})"))
            for p in (50, 52, 54, 56):  # team votes: the skip rate is a steep function of p
                out.append(("kmeans", wl, f"perfo(random:{p}) {S['kmeans']} level(team)"))
            for kind, arg in (("small", 2), ("small", 4), ("large", 2)):
                out.append(("kmeans", wl, f"perfo({kind}:{arg}) {S['kmeans']}"))
    if "lavamd" in apps:
        wl = dict(n=0, ipt=1, boxes1d=32 if quick else 48)
        for lv in ("thread", "warp", "team"):
            for h, p, thr in ((1, 1, 0.5), (2, 1, 0.1), (2, 2, 0.1), (3, 8, 0.1), (2, 4, 0.2), (3, 2, 0.5)):
                out.append(("lavamd", wl, f"memo(out:{h}:{p}:{thr}) {S['lavamd']} level({lv})"))
        for kind, arg in (("small", 4), ("herded_small", 4), ("random", 25)):
            out.append(("lavamd", wl, f"perfo({kind}:{arg}) {S['lavamd']} level(warp)"))
    return out


def point_key(app, wl, directive):
    return json.dumps([app, sorted(wl.items()), directive])


def load_done(part: Path):
    done = {}
    if part.exists():
        for line in part.read_text().splitlines():
            if not line.strip():
                continue
            key, row = line.split("\t", 1)
            done[key] = row
    return done


def merge(out: Path, parts, meta):
    rows = {}
    for p in parts:
        for k, r in load_done(p).items():
            rows[k] = r
    recs = sorted((T.from_csv_row(r) for r in rows.values()), key=lambda r: r.sort_key())
    tmp = out.with_suffix(out.suffix + ".tmp")
    tmp.write_text(T.HEADER + "\n" + "".join(T.to_csv_row(r) + "\n" for r in recs))
    os.replace(tmp, out)  # atomic (sweep.hpp:275-282)
    out.with_suffix(out.suffix + ".json").write_text(json.dumps(meta, indent=1))
    for p in parts:
        p.unlink(missing_ok=True)
    return recs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="sweep.csv")
    ap.add_argument("--apps", default="blackscholes,binomial,kmeans,lavamd")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--limit", type=int, default=0, help="only the first N points (smoke)")
    args = ap.parse_args()
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = Path(args.out)
    pts = points(args.apps.split(","), args.quick)
    if args.limit:
        pts = pts[: args.limit]
    part = Path(f"{out}.part.{rank}")
    done = {}
    for r in range(world):  # resume: points any rank already finished
        done.update(load_done(Path(f"{out}.part.{r}")))
    t0 = time.time()
    workloads = {}
    with part.open("a") as fh:
        for i, (app, wl, directive) in enumerate(pts):
            if i % world != rank:
                continue
            key = point_key(app, wl, directive)
            if key in done:
                continue
            wkey = json.dumps([app, sorted(wl.items())])
            if wkey not in workloads:
                workloads.clear()  # one resident workload per rank at a time
                torch.cuda.empty_cache()
                kw = {k: v for k, v in wl.items() if k not in ("n", "ipt")}
                workloads[wkey] = T.make_workload(app, wl["n"], wl["ipt"], **kw)
            rec = T.run_trial(workloads[wkey], directive)
            fh.write(key + "\t" + T.to_csv_row(rec) + "\n")
            fh.flush()
            print(f"[rank {rank}] {i + 1}/{len(pts)} {app} {rec.directive!r} {rec.status} "
                  f"speedup {rec.est_speedup:.3f} {rec.error_metric} {rec.error_value:.4g} "
                  f"rate {rec.approx_rate:.3f}", flush=True)
    if dist is not None:
        dist.barrier()
    if rank == 0:
        meta = {"points": len(pts), "world": world, "apps": args.apps, "quick": args.quick,
                "seconds": time.time() - t0, "device": torch.cuda.get_device_name(local),
                "columns": T.HEADER}
        recs = merge(out, [Path(f"{out}.part.{r}") for r in range(world)], meta)
        print(f"wrote {out} ({len(recs)} records)")
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
