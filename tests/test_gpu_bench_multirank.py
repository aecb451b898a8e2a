"""The N>1 path of bench.py (one process per GPU, barrier + max-over-ranks
timing, the K-Means all-reduce hook through torch.distributed) run as two
ranks on the one GPU this environment reaches (BENCH_DIST_BACKEND=gloo maps
both ranks onto cuda:0; the driver's scaling runs use NCCL, one GPU each)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("workload,port", [("blackscholes", 29621), ("kmeans", 29622)])
def test_bench_two_ranks(workload, port):
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--gpus", "2", "--workload", workload, "--steps", "1", "--warmup", "1", "--e2e-steps", "1",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["quality_ok"], lines[0][:3000]
