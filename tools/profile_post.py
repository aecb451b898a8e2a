#!/usr/bin/env python3
"""Reduce one profile round (tools/profile_round.sh TAG) to profiles/:
a summary table of every full capture (duration, DRAM bytes and GB/s, pipe
utilisation, warp execution efficiency, divergent branches, occupancy, top
stalls), SASS opcode histograms, the launch list, the bench lines, and the
`traffic` figures bench.py reports (profiles/traffic.json)."""
import csv
import gzip
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

CAPTURES = {  # capture name -> bench workload whose timed kernel it is
    "binomial_iact": "binomial-1M-x-1024-iact-team",
    "binomial_exact": None,
    "bs_taf": "blackscholes-4M-taf-h5",
    "bs_exact": None,
    "lavamd_taf": "lavamd-64^3-boxes-x-128-taf-warp",
    "lavamd_exact": None,
    "kmeans_region": "kmeans-lloyd-16M-x-32-x-64-perfo-random-team",
    "kmeans_update": None,
    "kmeans_compact": None,
}
METRICS = [
    ("duration_us", "gpu__time_duration.sum", 1e-3),
    ("dram_read_B", "dram__bytes_read.sum", 1),
    ("dram_write_B", "dram__bytes_write.sum", 1),
    ("dram_pct", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    ("fp64_pipe_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    ("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("dmma_pipe_pct", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
    ("issue_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("threads_per_inst", "smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    ("divergent_branch_targets", "smsp__sass_branch_targets_threads_divergent.sum", 1),
    ("occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("registers", "launch__registers_per_thread", 1),
]


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def read_raw(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    hdr, units = rows[0], rows[1]
    d = dict(zip(hdr, rows[2]))
    u = dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name", "?")}
    for key, metric, scale in METRICS:
        v = num(d.get(metric, ""))
        if v is not None:
            if metric.endswith("duration.sum"):
                v *= {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
                      "s": 1e9, "second": 1e9}.get(u.get(metric), 1.0)
            elif metric.startswith("dram__bytes") and u.get(metric) in ("Kbyte", "Mbyte", "Gbyte"):
                v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[metric]]
            out[key] = v * scale
    st = []
    for k in hdr:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            v = num(d.get(k, ""))
            if v:
                st.append((v, k[len("smsp__pcsamp_warps_issue_stalled_"):]))
    tot = sum(v for v, _ in st) or 1.0
    out["top_stalls"] = ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in sorted(st, reverse=True)[:4])
    return out


def main(tag):
    PROF.mkdir(exist_ok=True)
    lines = [f"# Profile round {tag} (B200, ncu --set full --clock-control none, one launch each)", "",
             "| capture | kernel | µs | DRAM MB (r+w) | DRAM GB/s | DRAM % | FP64 pipe % | DMMA pipe % | ALU % | issue % | "
             "warp exec eff | divergent branch targets | occupancy % | regs | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = json.loads((PROF / "traffic.json").read_text()) if (PROF / "traffic.json").exists() else {}
    for name, wl in CAPTURES.items():
        raw = OUT / f"{tag}_{name}_raw.csv"
        if not raw.exists():
            continue
        r = read_raw(raw)
        if r is None:
            continue
        byt = r.get("dram_read_B", 0) + r.get("dram_write_B", 0)
        us = r.get("duration_us") or 0
        gbs = byt / (us * 1e-6) / 1e9 if us else 0
        lines.append(f"| {name} | `{r['kernel'][:60]}` | {us:.1f} | {byt / 1e6:.1f} | {gbs:.0f} | "
                     f"{r.get('dram_pct', 0):.1f} | {r.get('fp64_pipe_pct', 0):.1f} | {r.get('dmma_pipe_pct', 0):.1f} | "
                     f"{r.get('alu_pipe_pct', 0):.1f} | "
                     f"{r.get('issue_pct', 0):.1f} | {r.get('threads_per_inst', 0) / 32:.3f} | "
                     f"{r.get('divergent_branch_targets', 0):.0f} | {r.get('occupancy_pct', 0):.1f} | "
                     f"{r.get('registers', 0):.0f} | {r['top_stalls']} |")
        if wl:
            traffic[wl] = int(byt)
        shutil.copy(OUT / f"{tag}_{name}_details.csv", PROF / f"{tag}_{name}_details.csv")
        with open(raw, "rb") as fi, gzip.open(PROF / f"{tag}_{name}_raw.csv.gz", "wb") as fo:
            fo.write(fi.read())
        src = OUT / f"{tag}_{name}_source.csv"
        if src.exists():
            h = subprocess.run([sys.executable, str(ROOT / "tools" / "sass_hist.py"), str(src)],
                               capture_output=True, text=True).stdout
            seen, keep = set(), []
            for ln in h.splitlines():
                if ln not in seen:
                    seen.add(ln)
                    keep.append(ln)
            (PROF / f"{tag}_{name}_sass_hist.txt").write_text("\n".join(keep) + "\n")
    lines += ["", "warp exec eff = thread instructions per warp instruction / 32 "
              "(smsp__thread_inst_executed_per_inst_executed.ratio)."]
    (PROF / f"{tag}_summary.md").write_text("\n".join(lines) + "\n")
    (PROF / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    for f in OUT.glob(f"{tag}_bench_*.json"):
        shutil.copy(f, PROF / f.name)
    for f in [OUT / f"{tag}_launches_binomial.csv", OUT / f"{tag}_gpu.txt"]:
        if f.exists():
            shutil.copy(f, PROF / f.name)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
