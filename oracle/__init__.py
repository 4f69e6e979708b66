"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for arXiv:1709.02599's counting.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_1709_02599_b200``) never imports it and shares no code
with it; both sides only share the seeded input generators in ``synth/``.

Two layers:

* ``dls_oracle.c`` (loaded through ctypes): the paper's nested-loop enumerator
  (Alg. 1/2) written with explicit row / column / diagonal scans over
  an int array, the Section 2.3 cell order, prefix (workunit)
  enumeration and square emission.
* pure Python below: the definitions of P:32 and P:521 (``is_latin``,
  ``is_diagonal``, ``is_vertically_symmetric``) and the row-permutation stacking
  brute force of Section 2.1, used only to pin the C oracle for N <= 5.

Pins: tests/test_oracle.py.  Every oracle function there is pinned against
something other than itself (brute force, the N! invariant, the VS definition
checked square by square, Fig. 1, the hourglass count of P:436, the DLS8 count of
P:476 through the prefix sum is GPU-only -- see DESIGN.md "Parity pins").
"""
from __future__ import annotations

import ctypes
import itertools
import math
import os
import subprocess
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dls_oracle.c")
_LIB = os.path.join(_HERE, "_dls_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile dls_oracle.c with gcc (plain C, no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        ip = ctypes.POINTER(ctypes.c_int)
        ull = ctypes.POINTER(ctypes.c_ulonglong)
        lib.oracle_count.argtypes = [ctypes.c_int, ctypes.c_int, ip, ip, ctypes.c_int, ull, ull]
        lib.oracle_count.restype = ctypes.c_int
        lib.oracle_count_levels.argtypes = [ctypes.c_int, ctypes.c_int, ip, ip, ctypes.c_int, ull, ull]
        lib.oracle_count_levels.restype = ctypes.c_int
        lib.oracle_prefixes.argtypes = [ctypes.c_int, ctypes.c_int, ip, ip, ctypes.c_int, ip, ctypes.c_longlong]
        lib.oracle_prefixes.restype = ctypes.c_longlong
        lib.oracle_squares.argtypes = [ctypes.c_int, ctypes.c_int, ip, ip, ctypes.c_int, ip, ctypes.c_longlong]
        lib.oracle_squares.restype = ctypes.c_longlong
        lib.oracle_plan.argtypes = [ctypes.c_int, ctypes.c_int, ip, ip]
        lib.oracle_plan.restype = ctypes.c_int
        lib.oracle_canonize.argtypes = [ctypes.c_int, ctypes.c_int, ip]
        lib.oracle_canonize.restype = ctypes.c_longlong
        lib.oracle_transform.argtypes = [ctypes.c_int, ip, ip, ctypes.c_int, ctypes.c_int, ip]
        lib.oracle_transform.restype = None
        llp = ctypes.POINTER(ctypes.c_longlong)
        lib.oracle_classes.argtypes = [ctypes.c_int, ctypes.c_int, ip, ip, ctypes.c_int, ip, llp,
                                       ctypes.c_longlong, llp]
        lib.oracle_classes.restype = ctypes.c_longlong
        _lib = lib
    return _lib


def _iarr(a) -> Tuple[np.ndarray, "ctypes._Pointer"]:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


# ---------------------------------------------------------------- grids

def empty_grid(n: int) -> np.ndarray:
    return np.full((n, n), -1, dtype=np.int32)


def first_row_grid(n: int) -> np.ndarray:
    """Row 0 fixed to 0..N-1 (normalisation)."""
    g = empty_grid(n)
    g[0, :] = np.arange(n)
    return g


# ---------------------------------------------------------------- plan

def plan(n: int, vs: bool = False, pre: Optional[np.ndarray] = None) -> List[int]:
    """Cell order of Section 2.3 for the cells not marked in ``pre``.

    ``pre`` is an n*n 0/1 array of cells assigned a priori; default = the fixed
    first row.  Returns cells as i*n+j.
    """
    if pre is None:
        pre = np.zeros((n, n), dtype=np.int32)
        pre[0, :] = 1
    pre_a, pre_p = _iarr(np.asarray(pre).reshape(-1) != 0)
    out, out_p = _iarr(np.zeros(n * n, dtype=np.int32))
    k = _load().oracle_plan(n, int(bool(vs)), pre_p, out_p)
    if k < 0:
        raise ValueError("oracle_plan failed: %d" % k)
    return [int(x) for x in out[:k]]


def plan_for_grid(n: int, vs: bool, grid: np.ndarray) -> List[int]:
    """Section 2.3 order of the empty cells of ``grid``."""
    return plan(n, vs, (np.asarray(grid).reshape(n, n) != -1).astype(np.int32))


# ---------------------------------------------------------------- counting

def count(n: int, vs: bool, grid: np.ndarray, order: Optional[Sequence[int]] = None) -> Tuple[int, int]:
    """(completions, nodes) of a partial square, cells filled in ``order``.

    Default order = the Section 2.3 order of the empty cells.  ``nodes`` is the
    number of consistent partial squares visited below ``grid`` ("node").
    """
    grid = np.asarray(grid).reshape(n, n)
    if order is None:
        order = plan_for_grid(n, vs, grid)
    g, gp = _iarr(grid.reshape(-1))
    o, op = _iarr(list(order) if len(order) else [0])
    c = ctypes.c_ulonglong(0)
    nd = ctypes.c_ulonglong(0)
    rc = _load().oracle_count(n, int(bool(vs)), gp, op, len(order), ctypes.byref(c), ctypes.byref(nd))
    if rc == -2:
        return 0, 0          # inconsistent partial square: nothing completes it
    if rc != 0:
        raise ValueError("oracle_count failed: %d" % rc)
    return int(c.value), int(nd.value)


def count_levels(n: int, vs: bool, grid: np.ndarray, order: Optional[Sequence[int]] = None) -> Tuple[int, List[int]]:
    """(completions, nodes per depth) of a partial square: entry k counts the
    consistent assignments of the first k+1 cells of ``order`` (R9, R15)."""
    grid = np.asarray(grid).reshape(n, n)
    if order is None:
        order = plan_for_grid(n, vs, grid)
    g, gp = _iarr(grid.reshape(-1))
    o, op = _iarr(list(order) if len(order) else [0])
    lv = (ctypes.c_ulonglong * max(len(order), 1))()
    c = ctypes.c_ulonglong(0)
    rc = _load().oracle_count_levels(n, int(bool(vs)), gp, op, len(order), ctypes.byref(c), lv)
    if rc == -2:
        return 0, [0] * len(order)
    if rc != 0:
        raise ValueError("oracle_count_levels failed: %d" % rc)
    return int(c.value), [int(lv[k]) for k in range(len(order))]


def count_all(n: int, vs: bool = False, fixed_first_row: bool = True) -> int:
    """Number of (VS)DLS of order n, optionally with row 0 = 0..N-1."""
    g = first_row_grid(n) if fixed_first_row else empty_grid(n)
    return count(n, vs, g)[0]


def prefixes(n: int, vs: bool, grid: np.ndarray, order: Sequence[int], depth: int,
             cap: Optional[int] = None) -> np.ndarray:
    """All consistent assignments of the first ``depth`` cells of ``order``."""
    lib = _load()
    g, gp = _iarr(np.asarray(grid).reshape(-1))
    o, op = _iarr(list(order) if len(order) else [0])
    if cap is None:
        cap = lib.oracle_prefixes(n, int(bool(vs)), gp, op, depth, None, 0)
        if cap < 0:
            raise ValueError("oracle_prefixes failed: %d" % cap)
    out = np.zeros((max(cap, 1), n * n), dtype=np.int32)
    total = lib.oracle_prefixes(n, int(bool(vs)), gp, op, depth,
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), cap)
    if total < 0:
        raise ValueError("oracle_prefixes failed: %d" % total)
    return out[:min(total, cap)].reshape(-1, n, n)


def count_prefixes(n: int, vs: bool, grid: np.ndarray, order: Sequence[int], depth: int) -> int:
    lib = _load()
    g, gp = _iarr(np.asarray(grid).reshape(-1))
    o, op = _iarr(list(order) if len(order) else [0])
    total = lib.oracle_prefixes(n, int(bool(vs)), gp, op, depth, None, 0)
    if total < 0:
        raise ValueError("oracle_prefixes failed: %d" % total)
    return int(total)


def squares(n: int, vs: bool, grid: np.ndarray, order: Optional[Sequence[int]] = None,
            cap: int = 1 << 20) -> np.ndarray:
    """Every completion of ``grid`` as full n x n arrays (up to ``cap``)."""
    grid = np.asarray(grid).reshape(n, n)
    if order is None:
        order = plan_for_grid(n, vs, grid)
    g, gp = _iarr(grid.reshape(-1))
    o, op = _iarr(list(order) if len(order) else [0])
    out = np.zeros((cap, n * n), dtype=np.int32)
    total = _load().oracle_squares(n, int(bool(vs)), gp, op, len(order),
                                   out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), cap)
    if total < 0:
        raise ValueError("oracle_squares failed: %d" % total)
    if total > cap:
        raise ValueError("more than cap=%d squares" % cap)
    return out[:total].reshape(-1, n, n)


# ---------------------------------------------------------------- definitions

def is_latin(sq: np.ndarray) -> bool:
    """Every row and every column holds each of 0..N-1 exactly once."""
    sq = np.asarray(sq)
    n = sq.shape[0]
    want = list(range(n))
    return all(sorted(sq[i, :].tolist()) == want for i in range(n)) and \
        all(sorted(sq[:, j].tolist()) == want for j in range(n))


def is_diagonal(sq: np.ndarray) -> bool:
    """Latin, and both the main diagonal and the main antidiagonal hold every element."""
    sq = np.asarray(sq)
    n = sq.shape[0]
    want = list(range(n))
    return is_latin(sq) and sorted(sq[k, k] for k in range(n)) == want and \
        sorted(sq[k, n - 1 - k] for k in range(n)) == want


def is_vertically_symmetric(sq: np.ndarray) -> bool:
    """LS[i][j] = N-1-LS[i][N-1-j] for all i, j."""
    sq = np.asarray(sq)
    n = sq.shape[0]
    return all(int(sq[i, j]) + int(sq[i, n - 1 - j]) == n - 1 for i in range(n) for j in range(n))


# ---------------------------------------------------------------- brute force (Section 2.1)

def brute_force_squares(n: int, diagonal: bool = True, vs: bool = False,
                        fixed_first_row: bool = True) -> List[np.ndarray]:
    """Stack rows chosen from all N! permutations: a row is kept when it
    has no equal element in the same position as an earlier row; complete
    stackings are then filtered by the definitions.  For N <= 5 only."""
    if n > 5:
        raise ValueError("brute force is for N <= 5")
    perms = list(itertools.permutations(range(n)))
    pa = np.array(perms, dtype=np.int32).reshape(len(perms), n)
    # compatible[a, b]: rows a and b have no equal element in the same position
    compatible = ~(pa[:, None, :] == pa[None, :, :]).any(axis=2)
    first = [perms.index(tuple(range(n)))] if fixed_first_row else range(len(perms))
    found: List[np.ndarray] = []

    def rec(rows: List[int], allowed: np.ndarray):
        if len(rows) == n:
            sq = pa[rows]
            if diagonal and not is_diagonal(sq):
                return
            if vs and not is_vertically_symmetric(sq):
                return
            found.append(sq.copy())
            return
        for p in np.nonzero(allowed)[0]:
            rec(rows + [int(p)], allowed & compatible[p])

    for f in first:
        rec([f], compatible[f].copy())
    return found


def brute_force_count(n: int, diagonal: bool = True, vs: bool = False,
                      fixed_first_row: bool = True) -> int:
    return len(brute_force_squares(n, diagonal, vs, fixed_first_row))


def vs_first_row_multiplier(n: int) -> int:
    """Number of vertically symmetric first rows: (N/2)! * 2^(N/2) for even N
    (reading R3).  Pinned in tests against brute force."""
    if n % 2:
        return 0
    return math.factorial(n // 2) * 2 ** (n // 2)


# ---------------------------------------------------------------- symmetry breaking (Section 4)

def hourglass_cells(n: int) -> List[int]:
    """Cells of a hourglass design other than row 0: both diagonals, then
    row N-1, each in row-major order."""
    diag = [i * n + j for i in range(1, n) for j in range(n) if i == j or i + j == n - 1]
    last = [(n - 1) * n + j for j in range(n) if (n - 1) * n + j not in diag]
    return diag + last


def hourglasses(n: int, vs: bool = False) -> np.ndarray:
    """All hourglass designs with row 0 = 0..N-1 (oracle prefix enumeration)."""
    cells = hourglass_cells(n)
    if vs:
        cells = [c for c in cells if 2 * (c % n) <= n - 1]
    return prefixes(n, vs, first_row_grid(n), cells, len(cells))


def canonize(n: int, vs: bool, grid: np.ndarray) -> int:
    """Alg. 5: 0 if ``grid`` is not the canonic form of its class,
    else the number of distinct designs in its class."""
    g, gp = _iarr(np.asarray(grid).reshape(-1))
    return int(_load().oracle_canonize(n, int(bool(vs)), gp))


def hourglass_classes(n: int, vs: bool = False, keep: bool = True):
    """Canonic hourglass designs and their class sizes (Alg. 5/6).
    Returns (reps (k, n, n) int32, mult (k,) int64, n_hourglasses), or with
    keep=False (number of classes, None, n_hourglasses) from a single pass."""
    lib = _load()
    cells = hourglass_cells(n)
    if vs:
        cells = [c for c in cells if 2 * (c % n) <= n - 1]
    g, gp = _iarr(first_row_grid(n).reshape(-1))
    o, op = _iarr(cells)
    nd = ctypes.c_longlong(0)
    llp = ctypes.POINTER(ctypes.c_longlong)
    k = lib.oracle_classes(n, int(bool(vs)), gp, op, len(cells), None, None, 0, ctypes.byref(nd))
    if k < 0:
        raise ValueError("oracle_classes failed: %d" % k)
    if not keep:
        return int(k), None, int(nd.value)
    reps = np.zeros((max(k, 1), n * n), dtype=np.int32)
    mult = np.zeros(max(k, 1), dtype=np.int64)
    lib.oracle_classes(n, int(bool(vs)), gp, op, len(cells), reps.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                       mult.ctypes.data_as(llp), k, ctypes.byref(nd))
    return reps[:k].reshape(-1, n, n), mult[:k], int(nd.value)


def transform(n: int, grid: np.ndarray, pi: Sequence[int], swap: int, mirror: bool) -> np.ndarray:
    """Image of a (partial) square under one M-transformation, renamed so that row
    0 reads 0..N-1."""
    g, gp = _iarr(np.asarray(grid).reshape(-1))
    p_, pp = _iarr(list(pi))
    out = np.zeros(n * n, dtype=np.int32)
    _load().oracle_transform(n, gp, pp, int(swap), int(bool(mirror)), out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    return out.reshape(n, n)


def group_size(n: int, vs: bool = False) -> int:
    """2 * 2^h * (h-1)! transformations keep hourglass designs (Alg. 5 loop bounds,
    P:404-406); the mirror is neutralised for VS squares."""
    h = n // 2
    return (1 if vs else 2) * (2 ** h) * math.factorial(h - 1)
