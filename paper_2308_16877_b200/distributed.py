"""Multi-GPU host logic (one process per GPU, torch.distributed over NCCL).

* Option pricing / LavaMD shard trivially: each rank runs its own region over
  its own shard (weak scaling); only timing uses a collective.
* K-Means exchanges one packed [k*d sums | k counts | changed] buffer per Lloyd
  iteration (hpac_kmeans_problem_t.allreduce); `kmeans_allreduce_hook` builds
  that hook on top of torch.distributed (NCCL on GPUs, gloo on CPU tests).
"""
from __future__ import annotations

import os


def env():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, world: int, rank: int):
    """Contiguous shard [lo, hi) of n items for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def kmeans_allreduce_hook(group=None):
    """Sum the packed centroid partials across ranks (in place)."""
    import torch.distributed as dist

    def hook(buf):
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)

    return hook


def native_nccl_comm(rank: int, world: int):
    """The library's own NCCL communicator across the torch.distributed ranks
    (id broadcast over the default group), or None if NCCL is not loadable.
    Passed as kmeans_run(nccl_comm=...), the Lloyd loop's all-reduce runs
    inside its CUDA graph instead of a host callback per iteration."""
    import torch.distributed as dist

    from . import abi
    from . import engine as E
    if not abi.lib().hpac_nccl_available():
        return None
    obj = [E.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return E.nccl_comm_init_rank(world, obj[0], rank)


def max_over_ranks(values, device=None, group=None):
    """Element-wise max of a list of floats across ranks (device-timed numbers
    are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return list(values)
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()


def weak_scaling_value(items_per_rank: int, steps: int, total_ms_max: float, world: int) -> float:
    """Whole-job throughput: all ranks' items over the slowest rank's time."""
    return world * items_per_rank * steps / (total_ms_max * 1e-3)
