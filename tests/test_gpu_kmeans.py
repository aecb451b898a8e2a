"""K-Means Lloyd loop on the device vs the oracle's kmeans_benchmark
(bench/kmeans.hpp:62-144) and the reference's own kmeans tests."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from paper_2308_16877_b200 import abi
from paper_2308_16877_b200 import engine as E
from gpu_util import dev

pytestmark = pytest.mark.gpu


def _oracle_kmeans(pts, k, grid, spec, max_iters=40, seed_base=0):
    n, d = pts.shape
    assign = np.zeros(n, np.int32)
    cent = np.zeros((k, d))
    it, conv = np.zeros(1, np.int32), np.zeros(1, np.int32)
    import ctypes as C
    st = abi.Stats()
    err = C.create_string_buffer(512)
    it_c, conv_c = C.c_int32(), C.c_int32()
    rc = oracle.oracle().oracle_kmeans_benchmark(pts.ctypes.data, n, d, k, C.byref(grid.c()),
                                                 C.byref(spec) if spec is not None else None,
                                                 max_iters, seed_base, assign.ctypes.data, cent.ctypes.data,
                                                 C.byref(it_c), C.byref(conv_c), C.byref(st), err, 512)
    assert rc == 0, err.value
    return assign, cent, it_c.value, bool(conv_c.value), st


@pytest.mark.parametrize("n,d,k,sep,spec_fn", [
    (512, 2, 4, 14.0, lambda: None),
    (4096, 2, 8, 8.0, lambda: None),
    (4096, 8, 16, 8.0, lambda: None),
    (8192, 32, 64, 30.0, lambda: None),
    (4096, 2, 8, 8.0, lambda: E.perfo("small", 4)),
    (4096, 2, 8, 8.0, lambda: E.perfo("large", 2)),
    (4096, 4, 8, 8.0, lambda: E.perfo("random", 20)),
    (4096, 2, 8, 8.0, lambda: E.iact(4, 0.0, 1)),
])
def test_lloyd_matches_oracle(n, d, k, sep, spec_fn):
    pts = E.make_blobs(n, d, k, 3, sep)
    grid, _ = E.resolve_grid("kmeans", n)
    r = E.kmeans_run(grid, dev(pts), k, spec_fn(), max_iters=40, perfo_seed_base=11)
    a, c, it, conv, st = _oracle_kmeans(pts, k, grid, spec_fn(), 40, 11)
    assert r.iterations == it and r.converged == conv
    assert r.stats["total_invocations"] == st.total_invocations
    assert r.stats["approx_invocations"] == st.approx_invocations
    ga = r.assignments.cpu().numpy()
    mcr = float(np.mean(ga != a))
    assert mcr <= 1e-3, mcr  # centroid sums differ in summation order only
    if mcr == 0:
        assert np.allclose(r.centroids.cpu().numpy(), c, rtol=1e-12, atol=1e-12)


def test_separable_converges_fast():
    """test_bench.cpp:139-163"""
    pts = E.make_blobs(512, 2, 4, 11, 14.0)
    grid = E.GridConfig(2, 64, 32, 4)
    r = E.kmeans_run(grid, dev(pts), 4)
    assert r.converged and r.iterations <= 2
    lab = r.assignments.cpu().numpy()
    mapping = {}
    for i, l in enumerate(lab):
        assert mapping.setdefault(i % 4, l) == l


def test_iact_threshold_zero_exact_assignments():
    """test_bench.cpp:165-185"""
    pts = E.make_blobs(512, 2, 4, 3, 8.0)
    grid = E.GridConfig(2, 64, 32, 4)
    acc = E.kmeans_run(grid, dev(pts), 4)
    app = E.kmeans_run(grid, dev(pts), 4, E.iact(4, 0.0))
    assert E.mcr(acc.assignments, app.assignments) == 0.0
    assert app.iterations == acc.iterations


def test_allreduce_hook_two_identical_shards():
    """Multi-GPU plumbing: an all-reduce that sums two identical shards must
    leave centroids, labels and iterations unchanged (sums and counts double)."""
    pts = E.make_blobs(4096, 4, 8, 5, 8.0)
    grid, _ = E.resolve_grid("kmeans", 4096)
    single = E.kmeans_run(grid, dev(pts), 8)
    calls = []

    def doubled(buf):
        calls.append(1)
        buf.mul_(2.0)

    twice = E.kmeans_run(grid, dev(pts), 8, allreduce=doubled)
    assert len(calls) == twice.iterations == single.iterations
    assert torch.equal(single.assignments, twice.assignments)
    assert torch.allclose(single.centroids, twice.centroids, rtol=0, atol=0)


def test_native_nccl_allreduce_hook():
    """hpac_nccl_allreduce as the Lloyd loop's all-reduce hook (single-rank
    NCCL communicator: the sum over one rank is the identity, so the run must
    equal the hook-less one bit for bit)."""
    if not abi.lib().hpac_nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    pts = E.make_blobs(8192, 8, 16, 9, 30.0)
    grid, _ = E.resolve_grid("kmeans", 8192)
    comm = E.nccl_comms(1)[0]
    try:
        a = E.kmeans_run(grid, dev(pts), 16, E.perfo("random", 25, seed=3), max_iters=20, perfo_seed_base=5)
        b = E.kmeans_run(grid, dev(pts), 16, E.perfo("random", 25, seed=3), max_iters=20, perfo_seed_base=5,
                         nccl_comm=comm)
        # the hook inside the captured loop (or its host-loop fallback) and
        # the host-driven loop agree
        c = E.kmeans_run(grid, dev(pts), 16, E.perfo("random", 25, seed=3), max_iters=20, perfo_seed_base=5,
                         nccl_comm=comm, host_loop=True)
    finally:
        abi.lib().hpac_nccl_comm_destroy(C.c_void_p(comm))
    print("nccl hook captured in the graph:", b.graph)
    for r in (b, c):
        assert a.iterations == r.iterations
        assert torch.equal(a.assignments, r.assignments) and torch.equal(a.centroids, r.centroids)


@pytest.mark.parametrize("n,d,k,sep,spec_fn,iters", [
    (8192, 32, 64, 30.0, lambda: None, 40),
    (8192, 32, 64, 8.0, lambda: None, 7),
    (4096, 2, 8, 8.0, lambda: E.perfo("small", 4), 40),
    (8192, 32, 64, 30.0, lambda: E.perfo("random", 52, level="team"), 40),
    (8192, 32, 64, 8.0, lambda: E.perfo("random", 30, level="warp"), 12),
    (4096, 2, 8, 8.0, lambda: E.iact(4, 0.0, 1), 40),
    (512, 2, 4, 14.0, lambda: None, 1),
])
def test_graph_loop_equals_host_loop(n, d, k, sep, spec_fn, iters):
    """The CUDA-graph Lloyd loop (conditional WHILE node, device-side
    convergence, device perforation seed) runs the same kernels in the same
    order as the host-driven loop: identical labels, centroids (bitwise),
    iteration count, convergence and stats."""
    pts = dev(E.make_blobs(n, d, k, 5, sep))
    grid, _ = E.resolve_grid("kmeans", n)
    g = E.kmeans_run(grid, pts, k, spec_fn(), max_iters=iters, perfo_seed_base=3)
    h = E.kmeans_run(grid, pts, k, spec_fn(), max_iters=iters, perfo_seed_base=3, host_loop=True)
    assert g.graph and not h.graph
    assert (g.iterations, g.converged) == (h.iterations, h.converged)
    assert torch.equal(g.assignments, h.assignments)
    assert torch.equal(g.centroids, h.centroids)
    for key in ("total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps"):
        assert g.stats[key] == h.stats[key], key
    assert g.region_ms > 0 and g.update_ms > 0


def test_native_nccl_comm_init_rank_single_process():
    """hpac_nccl_unique_id + hpac_nccl_comm_init_rank (the multi-process
    communicator bench.py uses under torchrun) with one rank: the Lloyd
    loop with its all-reduce captured in the graph equals the hook-less run."""
    if not abi.lib().hpac_nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    uid = E.nccl_unique_id()
    assert len(uid) == 128
    comm = E.nccl_comm_init_rank(1, uid, 0)
    pts = E.make_blobs(8192, 32, 64, 4, 30.0)
    grid, _ = E.resolve_grid("kmeans", 8192)
    try:
        a = E.kmeans_run(grid, dev(pts), 64, E.perfo("random", 40, level="team"), max_iters=15, perfo_seed_base=2)
        b = E.kmeans_run(grid, dev(pts), 64, E.perfo("random", 40, level="team"), max_iters=15, perfo_seed_base=2,
                         nccl_comm=comm)
    finally:
        abi.lib().hpac_nccl_comm_destroy(C.c_void_p(comm))
    assert b.graph
    assert a.iterations == b.iterations
    assert torch.equal(a.assignments, b.assignments) and torch.equal(a.centroids, b.centroids)


@pytest.mark.parametrize("host_loop", [False, True])
def test_lloyd_run_to_run_deterministic(host_loop):
    """Incremental centroid sums with fixed-order reductions: two runs on the
    same inputs give bitwise-identical centroids, labels and stats."""
    pts = dev(E.make_blobs(40000, 32, 64, 8, 12.0))
    grid, _ = E.resolve_grid("kmeans", 40000)
    spec = E.perfo("random", 40, level="warp")
    runs = [E.kmeans_run(grid, pts, 64, spec, max_iters=25, perfo_seed_base=9, host_loop=host_loop)
            for _ in range(2)]
    a, b = runs
    assert a.iterations == b.iterations and a.converged == b.converged
    assert torch.equal(a.assignments, b.assignments)
    assert torch.equal(a.centroids, b.centroids)
    for key in ("total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps"):
        assert a.stats[key] == b.stats[key], key


@pytest.mark.parametrize("host_loop", [False, True])
def test_lloyd_empty_cluster_keeps_centroid(host_loop):
    """Duplicate initial centroids: ties go to the lower index, so the
    duplicate's cluster starts empty and keeps its centroid (kmeans.hpp:142-143);
    later it refills from running sums that restarted from zero."""
    n, d, k = 8192, 32, 16
    pts = E.make_blobs(n, d, k, 21, 10.0)
    pts[3] = pts[1]  # Forgy init = first k points: centroid 3 duplicates centroid 1
    grid, _ = E.resolve_grid("kmeans", n)
    # iteration 1: cluster 3 is empty and keeps its centroid
    r1 = E.kmeans_run(grid, dev(pts), k, None, max_iters=1, host_loop=host_loop)
    assert not np.any(r1.assignments.cpu().numpy() == 3)
    assert np.array_equal(r1.centroids.cpu().numpy()[3], pts[3])
    # the full run (cluster 3 refills once centroid 1 moves: the running sums
    # restart from zero) matches the oracle's full re-sums
    r = E.kmeans_run(grid, dev(pts), k, None, max_iters=30, host_loop=host_loop)
    a, c, it, conv, st = _oracle_kmeans(pts, k, grid, None, 30, 0)
    assert r.iterations == it and r.converged == conv
    ga = r.assignments.cpu().numpy()
    mcr = float(np.mean(ga != a))
    assert mcr <= 1e-3
    if mcr == 0:
        assert np.allclose(r.centroids.cpu().numpy(), c, rtol=1e-12, atol=1e-12)


def test_failing_python_hook_raises():
    """A Python all-reduce hook that raises must stop the Lloyd loop with an
    error (the exception cannot cross the C boundary; it is re-raised), not
    continue on this rank's un-reduced partials."""
    pts = E.make_blobs(2048, 4, 8, 5, 8.0)
    grid, _ = E.resolve_grid("kmeans", 2048)

    def broken(buf):
        raise RuntimeError("peer lost")

    with pytest.raises(E.CudaError, match="peer lost"):
        E.kmeans_run(grid, dev(pts), 8, allreduce=broken)


def test_hook_nonzero_status_is_an_error():
    """hpac_allreduce_fn returning nonzero -> HPAC_ERR_CUDA from hpac_kmeans_run
    (host loop and graph capture alike), with the failing status in the message."""
    pts = dev(E.make_blobs(2048, 4, 8, 5, 8.0))
    n, d, k = 2048, 4, 8
    grid, _ = E.resolve_grid("kmeans", n)
    calls = []

    @abi.ALLREDUCE_FN
    def failing(buf, count, user, st):
        calls.append(count)
        return 7

    for flags in (0, abi.KMEANS_HOST_LOOP):
        cent = torch.empty((k, d), dtype=torch.float64, device="cuda")
        assign = torch.empty(n, dtype=torch.int32, device="cuda")
        pb = abi.KmeansProblem()
        pb.n_points, pb.dims, pb.k = n, d, k
        pb.points, pb.centroids, pb.assignments = pts.data_ptr(), cent.data_ptr(), assign.data_ptr()
        pb.max_iters, pb.flags = 10, flags
        pb.allreduce = failing
        res = abi.KmeansResult()
        err = C.create_string_buffer(512)
        rc = abi.lib().hpac_kmeans_run(C.byref(grid.c()), C.byref(pb), None, None, C.byref(res), err, 512)
        assert rc == abi.ERR_CUDA, (rc, err.value)
        assert b"status 7" in err.value
    assert calls and all(c == k * d + k + 1 for c in calls)


def test_nccl_hook_without_communicator_is_an_error():
    rc = abi.lib().hpac_nccl_allreduce(None, 0, None, None)
    assert rc in (abi.ERR_UNSUPPORTED,)


def test_lloyd_cluster_losing_half_its_points():
    """Regression for the running-sum update (kmeans_accumulate): with k*d + k
    > 256 the update spans several CTAs, and a cluster that loses at least half
    of its points in one iteration must keep correct sums (it did not when a
    sum thread could read the already-updated count). Forgy init on a
    adversarial point order: the first k points all sit in one blob, so the
    first iterations move most points between clusters."""
    n, d, k = 8192, 32, 64
    pts = E.make_blobs(n, d, k, 11, 30.0)
    order = np.argsort(np.arange(n) % k, kind="stable")  # blob 0's points first
    pts = np.ascontiguousarray(pts[order])
    grid, _ = E.resolve_grid("kmeans", n)
    want_a, want_c, want_it, want_conv, _ = _oracle_kmeans(pts, k, grid, None, 40)
    for host_loop in (False, True):
        for _ in range(3):
            r = E.kmeans_run(grid, dev(pts), k, max_iters=40, host_loop=host_loop)
            assert r.iterations == want_it and r.converged == want_conv
            mcr = float((r.assignments.cpu().numpy() != want_a).mean())
            assert mcr <= 1e-3, mcr
            assert np.allclose(r.centroids.cpu().numpy(), want_c, rtol=1e-9, atol=1e-9)


def test_python_hook_on_a_non_current_stream():
    """kmeans_run on a stream that is not torch's current stream: the hook's
    collective (ordered by torch against its current stream) must still see
    the finished partials and be seen by the library's readback (ADVICE r01:
    stream ordering of the torch.distributed hook)."""
    pts = E.make_blobs(8192, 8, 16, 5, 12.0)
    grid, _ = E.resolve_grid("kmeans", 8192)
    single = E.kmeans_run(grid, dev(pts), 16, host_loop=True)
    side = torch.cuda.Stream()

    def doubled(buf):
        torch.cuda._sleep(2_000_000)  # a slow collective on torch's current stream
        buf.mul_(2.0)

    r = E.kmeans_run(grid, dev(pts), 16, allreduce=doubled, stream=side)
    torch.cuda.synchronize()
    assert r.iterations == single.iterations
    assert torch.equal(r.assignments, single.assignments)
    assert torch.equal(r.centroids, single.centroids)
