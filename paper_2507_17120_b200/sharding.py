"""Data-parallel sharding of a window across GPUs.

Requests are independent given the bucket edges, and the edges depend only on
the global length histogram (BucketSet.adjust_buckets reads counts,
bucket_manager.py:133-191; current_n_max reads N and sum(len),
batch_controller.py:93-104).  So a window of N requests is split into contiguous
arrival-order shards, one per rank; each rank builds its local histogram (K1),
the histograms are summed with one all-reduce (C1, NCCL over NVLink/NVSwitch on
the GPU box; gloo in the CPU tests), every rank derives identical edges from the
global histogram (K2), and order / size / pack stay shard-local.
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[start, end) of rank's contiguous arrival-order shard of an n-request window."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    return rank * n // world, (rank + 1) * n // world


def allreduce_histogram(hist, group=None):
    """C1: in-place sum of the per-rank (class, length) histograms.  The counts are
    int32 (bit patterns of the uint32 counters; N < 2^31 per window), so the sum is
    exact integer arithmetic on every backend."""
    import torch.distributed as dist
    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist
