"""Multi-GPU plumbing for the batch-sharded protected convolution.

The path shards naturally: images are independent, and by linearity every
per-shard FIC / IC / ICBatch check is an exact restriction of the global check.
The only collective is one tiny integer all-reduce (error counts, campaign class
counts) over NCCL/NVLink -- or gloo for the CPU tests.  Campaign trials shard by
trial index; trial seeds derive_seed(root, t) do not depend on the GPU count,
so the folded report is identical for any world size.
"""
from __future__ import annotations

import torch


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of `total` items for `rank` (balanced to +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return total * rank // world, total * (rank + 1) // world


def allreduce_counts(counts, device=None) -> list[int]:
    """Sum small integer vectors (verdict / campaign counts) over all ranks."""
    import torch.distributed as dist
    t = torch.as_tensor(list(counts), dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
    return [int(v) for v in t.tolist()]


def max_over_ranks(value: float, device=None) -> float:
    """Multi-GPU timing rule: the step time is the slowest rank's."""
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sharded_campaign(run_range, trials: int, rank: int, world: int, device=None) -> list[int]:
    """run_range(begin, end) -> (detected, benign, sdc, masked) for this rank's trial
    shard; returns the global report counts."""
    b, e = shard_range(trials, rank, world)
    return allreduce_counts(run_range(b, e), device=device)
