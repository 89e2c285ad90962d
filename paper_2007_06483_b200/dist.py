"""Multi-GPU batch sharding: independent pairs/stacks are
split across ranks with no collective on the data path; the only
communication is the start/stop barrier and the max-over-ranks time.

One process per GPU (torchrun); NCCL on GPUs, gloo in the CPU tests.
"""

from __future__ import annotations


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) slice of n_items for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(n_items, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def shard_pairs(pairs: list, rank: int, world: int) -> list:
    b, e = shard_range(len(pairs), rank, world)
    return pairs[b:e]


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (the job's time is its slowest rank)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
