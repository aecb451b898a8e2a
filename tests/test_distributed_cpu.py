"""World-size-2 gloo tests of the multi-GPU host logic (no GPU needed):
the K-Means partial-sum exchange protocol, max-over-ranks timing and shard
bounds, plus bench.py's reference arm under torchrun."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _lloyd_shard(rank, world, port, pts, k, iters, q):
    """One rank of a sharded Lloyd loop: region on the shard (oracle), packed
    partials, all-reduce hook (product code), centroid recompute."""
    sys.path.insert(0, str(ROOT))
    import oracle
    from paper_2308_16877_b200 import distributed as D
    from paper_2308_16877_b200 import engine as E
    _init(rank, world, port)
    n, d = pts.shape
    lo, hi = D.shard_range(n, world, rank)
    mine = np.ascontiguousarray(pts[lo:hi])
    cent = pts[:k].copy()  # Forgy on the global first k points
    assign = np.full(hi - lo, -1, np.int32)
    dist_label = np.zeros(hi - lo, np.int32)
    hook = D.kmeans_allreduce_hook()
    grid = E.GridConfig(max(1, -(-(hi - lo) // 256)), 64, 32, 4)
    it_done = 0
    for it in range(1, iters + 1):
        rc, st, msg = oracle.oracle_run(grid, hi - lo, 0, E.kmeans_region(mine, cent, dist_label), None)
        assert rc == 0, msg
        buf = np.zeros(k * d + k + 1)
        for i, c in enumerate(dist_label):
            buf[c * d:(c + 1) * d] += mine[i]
            buf[k * d + c] += 1
            if assign[i] != c:
                buf[-1] += 1
                assign[i] = c
        t = torch.from_numpy(buf)
        hook(t)
        it_done = it
        if t[-1].item() == 0:
            break
        red = t.numpy()
        for c in range(k):
            if red[k * d + c] > 0:
                cent[c] = red[c * d:(c + 1) * d] / red[k * d + c]
    q.put((rank, lo, assign.copy(), cent.copy(), it_done))
    dist.destroy_process_group()


def test_sharded_lloyd_protocol_matches_single_process():
    sys.path.insert(0, str(ROOT))
    import oracle
    from paper_2308_16877_b200 import abi
    from paper_2308_16877_b200 import engine as E
    import ctypes as C
    pts = E.make_blobs(2000, 3, 5, 9, 12.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29511
    procs = [ctx.Process(target=_lloyd_shard, args=(r, 2, port, pts, 5, 20, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    labels = np.concatenate([r[2] for r in res])
    assert np.array_equal(res[0][3], res[1][3])  # identical centroids on every rank
    assert res[0][4] == res[1][4]
    # single-process reference Lloyd (oracle) on the whole problem
    a = np.zeros(2000, np.int32)
    it, cv = C.c_int32(), C.c_int32()
    st = abi.Stats()
    g = E.GridConfig(8, 64, 32, 4)
    rc = oracle.oracle().oracle_kmeans_benchmark(pts.ctypes.data, 2000, 3, 5, C.byref(g.c()), None, 20, 0,
                                                 a.ctypes.data, None, C.byref(it), C.byref(cv), C.byref(st),
                                                 None, 0)
    assert rc == 0
    assert np.array_equal(labels, a)
    assert res[0][4] == it.value


def _max_worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    from paper_2308_16877_b200 import distributed as D
    _init(rank, world, port)
    vals = D.max_over_ranks([10.0 * (rank + 1), 5.0 - rank])
    q.put((rank, vals))
    dist.destroy_process_group()


def test_max_over_ranks_and_weak_value():
    from paper_2308_16877_b200 import distributed as D
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_max_worker, args=(r, 2, 29512, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=60) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    for _, v in out:
        assert v == [20.0, 5.0]
    assert D.weak_scaling_value(1000, 2, 20.0, 2) == 2 * 1000 * 2 / 0.02


def test_shard_range_covers():
    from paper_2308_16877_b200 import distributed as D
    for n in (0, 1, 7, 1000, 1 << 20):
        for w in (1, 2, 3, 8):
            spans = [D.shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


@pytest.mark.slow
def test_bench_reference_arm_under_torchrun():
    """N=2: rank 0 alone runs the reference arm and prints; rank 1 exits 0."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29513", str(ROOT / "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--workload", "kmeans-region"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference"
