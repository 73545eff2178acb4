"""Right-hand-side sharding across ranks (one process per GPU).

The transform is applied column by column, so the multi-GPU path shards the RHS
batch over the ranks with the operator replicated and no collective on the data
path.  Only the timing uses a collective (max over ranks).  Host logic only; the
CPU tests exercise it with a gloo process group.
"""
from __future__ import annotations


def column_shard(B_total: int, rank: int, world: int) -> slice:
    """Columns [rank*B/G, (rank+1)*B/G) of a global batch of B_total (contiguous, balanced)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    lo = (B_total * rank) // world
    hi = (B_total * (rank + 1)) // world
    return slice(lo, hi)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks of the default process group (identity without one)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
