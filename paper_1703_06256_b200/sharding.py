"""Frame sharding across ranks: frames are independent, so each
rank runs its own pipeline over its own contiguous frame range and the data
path has no collective.  torch.distributed is used only to align the timed
region (barrier) and to take the slowest rank's time.
"""
from __future__ import annotations


def shard(rank: int, world: int, per_rank: int) -> range:
    """Weak scaling: rank r processes frames [r*per_rank, (r+1)*per_rank)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return range(rank * per_rank, (rank + 1) * per_rank)


def split(n: int, rank: int, world: int) -> range:
    """Strong scaling: a fixed batch of n frames split into contiguous shards
    whose sizes differ by at most one."""
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity when not
    distributed)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()
