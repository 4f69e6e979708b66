"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds none of the method's arithmetic (no cell order, no counting,
no candidate masks): it only draws random partial squares with the structure of
the paper's workunits -- first row fixed to 0..N-1 and both diagonals
assigned (the decomposition of P:481 puts the diagonals first, Fig. 1) -- and
rejects draws that break the uniqueness constraints among the given cells.

Grids are uint8 N x N arrays with EMPTY (=0xFF) for unassigned cells, the
record format of the C ABI (include/dls_b200.h).
"""
from __future__ import annotations

import numpy as np

EMPTY = 0xFF

# Fixed seeds of BASELINE.json's sampled configs.
SEED_VS10 = 1709        # config 4: 4096 vertically symmetric order-10 prefixes
SEED_DLS9 = 2599        # config 5: 1024 order-9 prefixes
N_VS10 = 4096
N_DLS9 = 1024


def _consistent(g: np.ndarray) -> bool:
    """No value repeated among the assigned cells of a row, column, or diagonal."""
    n = g.shape[0]
    units = [g[i, :] for i in range(n)] + [g[:, j] for j in range(n)]
    units.append(np.array([g[k, k] for k in range(n)]))
    units.append(np.array([g[k, n - 1 - k] for k in range(n)]))
    for u in units:
        vals = u[u != EMPTY]
        if len(np.unique(vals)) != len(vals):
            return False
    return True


def diagonal_prefix(rng: np.random.Generator, n: int, max_tries: int = 10_000_000) -> np.ndarray:
    """First row 0..N-1, main diagonal and antidiagonal drawn uniformly among the
    consistent assignments (by rejection, BASELINE config 5): the main diagonal is
    a uniform permutation with LS[0][0]=0, the antidiagonal a uniform permutation
    with LS[0][N-1]=N-1, agreeing on the centre cell for odd N."""
    for _ in range(max_tries):
        md = np.concatenate([[0], 1 + rng.permutation(n - 1)])
        rest = np.array([v for v in range(n) if v != n - 1])
        ad = np.concatenate([[n - 1], rng.permutation(rest)])
        if n % 2 == 1 and md[n // 2] != ad[n // 2]:
            continue
        g = np.full((n, n), EMPTY, dtype=np.uint8)
        g[0, :] = np.arange(n)
        ok = True
        for k in range(1, n):
            for (i, j, v) in ((k, k, md[k]), (k, n - 1 - k, ad[k])):
                if g[i, j] != EMPTY and g[i, j] != v:
                    ok = False
                g[i, j] = v
        if ok and _consistent(g):
            return g
    raise RuntimeError("rejection sampling did not converge")


def vs_diagonal_prefix(rng: np.random.Generator, n: int, max_tries: int = 10_000_000) -> np.ndarray:
    """Vertically symmetric variant (BASELINE config 4): first row 0..N-1 (which
    satisfies LS[0][j] + LS[0][N-1-j] = N-1), main diagonal a uniform permutation
    with LS[0][0]=0, antidiagonal its mirror LS[i][N-1-i] = N-1-LS[i][i];
    rejected unless the given cells are consistent.  Even N only."""
    if n % 2:
        raise ValueError("vertically symmetric DLS need even N")
    for _ in range(max_tries):
        md = np.concatenate([[0], 1 + rng.permutation(n - 1)])
        g = np.full((n, n), EMPTY, dtype=np.uint8)
        g[0, :] = np.arange(n)
        for k in range(1, n):
            g[k, k] = md[k]
            g[k, n - 1 - k] = n - 1 - md[k]
        if _consistent(g):
            return g
    raise RuntimeError("rejection sampling did not converge")


def diagonal_prefixes(seed: int, n: int, count: int, vs: bool = False) -> np.ndarray:
    """``count`` independent draws from a fixed seed, shape (count, n, n) uint8."""
    rng = np.random.default_rng(seed)
    f = vs_diagonal_prefix if vs else diagonal_prefix
    return np.stack([f(rng, n) for _ in range(count)]) if count else np.zeros((0, n, n), np.uint8)


def to_int_grid(g: np.ndarray) -> np.ndarray:
    """uint8/EMPTY record -> int32 grid with -1 for empty (the oracle's format)."""
    a = np.asarray(g).astype(np.int32)
    a[a == EMPTY] = -1
    return a
