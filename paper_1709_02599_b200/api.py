"""User-level calls over the C ABI (marshalling only; the search is the CUDA kernel)."""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import _binding as B


def default_split_depth(n: int, symmetric: bool = False, fixed_first_row: bool = True) -> int:
    """Split at the diagonal depth: first row + both diagonals assigned (Fig. 1)."""
    return B.dls_plan(n, symmetric, fixed_first_row)[2]


def first_row_multiplier(n: int, symmetric: bool = False) -> int:
    """Full count / first-row-fixed count: N! for DLS, (N/2)!*2^(N/2) for
    vertically symmetric DLS (reading R3); computed by the library."""
    return B.dls_scale_total(n, 0, symmetric)[1]


def count_squares(n: int, symmetric: bool = False, fixed_first_row: bool = True,
                  depth: Optional[int] = None, stream: Optional[int] = None) -> dict:
    """Exhaustive count of (vertically symmetric) DLS of order n on the GPU."""
    d = default_split_depth(n, symmetric, fixed_first_row) if depth is None else depth
    pre = B.dls_split(n, d, symmetric, fixed_first_row)
    total, nodes = B.dls_count(n, d, pre, symmetric, fixed_first_row, stream=stream)
    out = {"n": n, "symmetric": symmetric, "fixed_first_row": fixed_first_row, "depth": d,
           "n_prefix": int(pre.shape[0]), "count": total, "nodes": nodes}
    if fixed_first_row:
        out["total_all_first_rows"] = B.dls_scale_total(n, total, symmetric)[0]
    return out


def count_prefixes(n: int, prefixes, symmetric: bool = False, fixed_first_row: bool = True,
                   depth: Optional[int] = None, stream: Optional[int] = None):
    """Per-prefix completion counts (uint64) of depth-`depth` records."""
    d = default_split_depth(n, symmetric, fixed_first_row) if depth is None else depth
    counts = np.zeros(int(prefixes.shape[0]), dtype=np.uint64)
    total, nodes = B.dls_count(n, d, prefixes, symmetric, fixed_first_row, out_counts=counts, stream=stream)
    return counts, total, nodes
