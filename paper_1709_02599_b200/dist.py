"""Multi-GPU plumbing: one process per GPU, workunits dealt round-robin.

The workunits of P:481 are independent ("embarrassing parallelism"), so
ranks exchange nothing while searching; the only collective is the final int64
sum of the counts.  ``torch.distributed`` is the plumbing (NCCL on B200s, gloo in
the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_workunits(records: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Round-robin share of rank ``rank``: records rank, rank+world, ...

    Round-robin (not contiguous blocks) because neighbouring workunits of the
    depth-first split have correlated subtree sizes."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return np.ascontiguousarray(records[rank::world])


def allreduce_count(value: int, device=None) -> int:
    """Sum an integer count over all ranks (int64; exact up to 9.2e18)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64, device=device)
    dist.all_reduce(t)
    return int(t.item())


def allreduce_max(value: float, device=None) -> float:
    """Max over ranks (the step time of a multi-GPU run is the slowest rank's)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
