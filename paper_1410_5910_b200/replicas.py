"""Multi-GPU execution: independent replicas, one process per GPU.

The online solve does not shard (the sweeps are a
dependency chain over layers and the north star fixes one GPU with no
collectives), so N GPUs run N replicas:
- each rank owns a disjoint subset of the right-hand sides;
- there is no collective on the data path;
- timing is bracketed by a barrier and reported as the max over ranks.

For the multi-RHS configuration (c5: 64 sources) the sources shard across
ranks; for a single-RHS workload every rank solves its own copy.
"""

from __future__ import annotations

import os

__all__ = ["world", "shard", "max_over_ranks", "gather_counts"]


def world():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_items: int, world_size: int, rank: int):
    """Contiguous, balanced index range of rank `rank` (first ranks take the remainder)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad world size / rank")
    base, rem = divmod(n_items, world_size)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return range(lo, hi)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. timed ms) over the process group, or itself."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_counts(count: int, device=None) -> int:
    """Sum of per-rank work counts (solves completed) over the process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return int(count)
    t = torch.tensor([int(count)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())
