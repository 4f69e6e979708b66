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


def shard_ranges(n_units: int, rank: int, world: int, chunk: int):
    """Round-robin share of rank ``rank`` of [0, n_units) cut into ``chunk``-sized
    ranges: [(begin, end), ...] for ranges rank, rank+world, ...  The diagonal
    workunits of the symmetry-broken search (dls_count_sb_range) are independent
    (P:483), and canonic designs cluster at small indices (symmetry
    breaking), so ranges are dealt round-robin rather than in blocks."""
    if world < 1 or not 0 <= rank < world or chunk < 1 or n_units < 0:
        raise ValueError("bad rank/world/chunk")
    starts = range(rank * chunk, n_units, world * chunk)
    return [(b, min(b + chunk, n_units)) for b in starts]


def count_sb_sharded(n: int, symmetric: bool, rank: int, world: int, chunk: int, n_units: int,
                     count_range=None, device=None) -> dict:
    """Alg. 6 over this rank's ranges, then one int64 all-reduce per total.
    ``count_range(n, begin, end, symmetric) -> dict(count, hourglasses, classes,
    nodes)`` defaults to the GPU call dls_count_sb_range."""
    if count_range is None:
        from ._binding import dls_count_sb_range

        def count_range(n_, b, e, vs):
            return dls_count_sb_range(n_, b, e, vs)
    local = {"count": 0, "hourglasses": 0, "classes": 0, "nodes": 0}
    for b, e in shard_ranges(n_units, rank, world, chunk):
        r = count_range(n, b, e, symmetric)
        for k in local:
            local[k] += int(r[k])
    out = {k: allreduce_count(v, device=device) for k, v in local.items()}
    out["local_count"] = local["count"]
    return out
