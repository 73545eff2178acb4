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


def rank_columns(B_global: int, rank: int, world: int, strong: bool = True) -> slice:
    """Columns of the config's seeded batch that rank `rank` applies: strong scaling (default) shards
    the global batch (column_shard); weak scaling gives every rank the whole batch (B per GPU fixed)."""
    return column_shard(B_global, rank, world) if strong else slice(0, B_global)


def relaunch_cmd(script: str, argv: list, gpus: int, port: int, python: str = "python") -> list:
    """`python bench.py --gpus N ...` started without a launcher: the same command under
    torch.distributed.run, one rank per GPU of this node (rendezvous on 127.0.0.1)."""
    return [python, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", script] + list(argv)


def world_from(env: dict, gpus: int):
    """(world_size, rank, local_rank, need_relaunch) from the launcher's environment and --gpus.
    A launcher-provided WORLD_SIZE must agree with --gpus when --gpus > 1."""
    ws = int(env.get("WORLD_SIZE", "0") or 0)
    if ws == 0:
        return (1, 0, 0, gpus > 1)
    if gpus > 1 and ws != gpus:
        raise ValueError(f"--gpus {gpus} but WORLD_SIZE={ws}")
    return (ws, int(env.get("RANK", "0")), int(env.get("LOCAL_RANK", "0")), False)
