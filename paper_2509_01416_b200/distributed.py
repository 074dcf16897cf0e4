"""Multi-GPU plumbing for the instance-parallel S_N solve: instances are independent,
so ranks shard the batch (or solve their own batch: weak scaling) with no data-path collective.
torch.distributed is used only for the barrier and the max/sum reductions of the timing."""
from __future__ import annotations

import os


def env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def rank_seed(rank: int, base: int = 2000) -> int:
    """Per-rank seed base for weak scaling: rank r solves instances seeded base + 100000 r + b."""
    return base + 100000 * rank


def shard(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous instance shard [begin, end) of rank (same partition rule as parallel.hpp:17-48)."""
    base, extra = divmod(n_items, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def reduce_max(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
