"""Thin ctypes binding of libdls_b200.so (argument marshalling only).

Names follow the C ABI in include/dls_b200.h.  Every step of the search runs in
the library's CUDA kernel; there is no Python or CPU fallback: on a machine
without a GPU ``dls_count`` raises ``DlsError(DLS_E_NODEVICE)``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

from . import build as _build

DLS_EMPTY = 0xFF
DLS_MAX_ORDER = 10
DLS_STATS_WORDS = 10
DLS_OK, DLS_E_ARG, DLS_E_CUDA, DLS_E_PREFIX, DLS_E_NODEVICE = 0, -1, -2, -3, -4

EXPORTS = ("dls_version", "dls_last_error", "dls_plan", "dls_split", "dls_refine", "dls_emit", "dls_count",
           "dls_count_async", "dls_canonize", "dls_count_sb", "dls_count_sb_range", "dls_count_cells",
           "dls_random_prefix", "dls_kernel_launches", "dls_search_levels", "dls_scale_total", "dls_mc_estimate")

_lib = None


class DlsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("%s (code %d)" % (msg, code))
        self.code = code


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load the in-tree library (building it first if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("DLS_LIB", _build.LIB)   # DLS_LIB: alternative build (tuning experiments)
    if path == _build.LIB and build_if_missing and (not os.path.exists(path) or _build._stale()):
        _build.build()
    if not os.path.exists(path):
        raise DlsError(DLS_E_NODEVICE, "libdls_b200.so is missing: run paper_1709_02599_b200.build")
    lib = ctypes.CDLL(path)
    c_int, c_i64, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
    lib.dls_version.restype = ctypes.c_char_p
    lib.dls_last_error.restype = ctypes.c_char_p
    lib.dls_plan.argtypes = [c_int, c_int, c_int, vp, vp, vp, vp]
    lib.dls_plan.restype = c_int
    lib.dls_split.argtypes = [c_int, c_int, c_int, c_int, vp, c_i64]
    lib.dls_split.restype = c_i64
    lib.dls_refine.argtypes = [c_int, c_int, c_int, c_int, vp, c_i64, c_int, vp, vp, c_i64]
    lib.dls_refine.restype = c_i64
    lib.dls_emit.argtypes = [c_int, c_int, c_int, c_int, vp, c_i64, vp, c_i64, vp]
    lib.dls_emit.restype = c_i64
    lib.dls_count.argtypes = [c_int, c_int, c_int, c_int, vp, c_i64, vp, vp, vp, vp]
    lib.dls_count.restype = c_int
    lib.dls_count_async.argtypes = [c_int, c_int, c_int, c_int, vp, c_i64, vp, vp, vp]
    lib.dls_count_async.restype = c_int
    lib.dls_canonize.argtypes = [c_int, c_int, vp, c_i64, vp, vp]
    lib.dls_canonize.restype = c_int
    lib.dls_count_sb.argtypes = [c_int, c_int, vp, vp, vp, vp, vp]
    lib.dls_count_sb.restype = c_int
    lib.dls_count_sb_range.argtypes = [c_int, c_int, c_i64, c_i64, vp, vp, vp, vp, vp]
    lib.dls_count_sb_range.restype = c_int
    lib.dls_count_cells.argtypes = [c_int, c_int, vp, vp, c_int, vp, vp, vp]
    lib.dls_count_cells.restype = c_int
    lib.dls_random_prefix.argtypes = [c_int, c_int, vp, vp, c_int, ctypes.c_uint64, vp, vp]
    lib.dls_random_prefix.restype = c_int
    lib.dls_kernel_launches.restype = c_int
    lib.dls_search_levels.argtypes = [c_int, c_int, c_int, c_int, vp]
    lib.dls_search_levels.restype = c_int
    lib.dls_scale_total.argtypes = [c_int, c_int, ctypes.c_uint64, vp, vp]
    lib.dls_scale_total.restype = c_int
    lib.dls_mc_estimate.argtypes = [vp, vp, c_i64, ctypes.c_double, vp]
    lib.dls_mc_estimate.restype = c_int
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc < 0:
        raise DlsError(int(rc), "%s: %s" % (what, load().dls_last_error().decode()))


def dls_version() -> str:
    return load().dls_version().decode()


def dls_plan(n: int, symmetric: bool = False, fixed_first_row: bool = True):
    """-> (cells[int32], forced[uint8], diag_depth)  (Section 2.3)."""
    cells = np.zeros(n * n, dtype=np.int32)
    forced = np.zeros(n * n, dtype=np.uint8)
    steps = ctypes.c_int32(0)
    dd = ctypes.c_int32(0)
    rc = load().dls_plan(n, int(symmetric), int(fixed_first_row), cells.ctypes.data, forced.ctypes.data,
                         ctypes.addressof(steps), ctypes.addressof(dd))
    _check(rc, "dls_plan")
    return cells[:steps.value].copy(), forced[:steps.value].copy(), int(dd.value)


def dls_split(n: int, depth: int, symmetric: bool = False, fixed_first_row: bool = True) -> np.ndarray:
    """All depth-`depth` prefix records, shape (count, n, n) uint8."""
    lib = load()
    total = lib.dls_split(n, int(symmetric), int(fixed_first_row), depth, None, 0)
    _check(total, "dls_split")
    out = np.empty((max(total, 1), n, n), dtype=np.uint8)
    got = lib.dls_split(n, int(symmetric), int(fixed_first_row), depth, out.ctypes.data, total)
    _check(got, "dls_split")
    return out[:total]


def dls_refine(n: int, depth: int, records: np.ndarray, depth2: int, symmetric: bool = False,
               fixed_first_row: bool = True):
    """Children of depth-`depth` records at depth2 -> (records (k, n, n) uint8, parent (k,) uint32)."""
    lib = load()
    recs = np.ascontiguousarray(records, dtype=np.uint8)
    total = lib.dls_refine(n, int(symmetric), int(fixed_first_row), depth, recs.ctypes.data, len(recs), depth2,
                           None, None, 0)
    _check(total, "dls_refine")
    out = np.empty((max(total, 1), n, n), dtype=np.uint8)
    par = np.empty(max(total, 1), dtype=np.uint32)
    got = lib.dls_refine(n, int(symmetric), int(fixed_first_row), depth, recs.ctypes.data, len(recs), depth2,
                         out.ctypes.data, par.ctypes.data, total)
    _check(got, "dls_refine")
    return out[:total], par[:total]


def _ptr(a) -> Tuple[int, object]:
    """(address, keepalive) of a numpy array or a torch tensor (host or CUDA)."""
    if a is None:
        return 0, None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data, a
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr(), a
    raise TypeError("expected numpy array or torch tensor")


def _dtype_name(a) -> str:
    return str(a.dtype).replace("torch.", "")


def _check_records(a, n: int, what: str) -> int:
    """Records must be uint8 of shape (k, n, n) (or (k, n*n)); returns k."""
    if a is None:
        return 0
    if _dtype_name(a) != "uint8":
        raise ValueError("%s: records must be uint8, got %s" % (what, _dtype_name(a)))
    shape = tuple(a.shape)
    if not (len(shape) == 3 and shape[1:] == (n, n)) and not (len(shape) == 2 and shape[1] == n * n):
        raise ValueError("%s: records must have shape (k, %d, %d), got %s" % (what, n, n, shape))
    return int(shape[0])


def _check_counts(c, k: int, what: str, device=None):
    """Per-prefix counts must be 8-byte integers with room for k entries."""
    if c is None:
        return
    if _dtype_name(c) not in ("uint64", "int64"):
        raise ValueError("%s: counts must be uint64/int64, got %s" % (what, _dtype_name(c)))
    if int(np.prod(tuple(c.shape))) < k:
        raise ValueError("%s: counts hold %d entries, need %d" % (what, int(np.prod(tuple(c.shape))), k))
    if device is not None and hasattr(c, "device") and str(c.device) != str(device):
        raise ValueError("%s: counts on %s but records on %s" % (what, c.device, device))


def dls_count(n: int, depth: int, prefixes, symmetric: bool = False, fixed_first_row: bool = True,
              out_counts=None, stream: Optional[int] = None) -> Tuple[int, int]:
    """Count completions of every prefix on the GPU -> (total, nodes).

    ``prefixes``: (count, n, n) uint8 records, numpy (host) or torch (host or cuda).
    ``out_counts``: optional uint64 numpy array / int64 torch tensor of length count.
    ``stream``: cudaStream_t handle (e.g. ``torch.cuda.current_stream().cuda_stream``).
    """
    n_prefix = _check_records(prefixes, n, "dls_count")
    _check_counts(out_counts, n_prefix, "dls_count")
    pp, keep1 = _ptr(prefixes)
    cp, keep2 = _ptr(out_counts)
    tot = ctypes.c_uint64(0)
    nodes = ctypes.c_uint64(0)
    rc = load().dls_count(n, int(symmetric), int(fixed_first_row), depth, pp or None, n_prefix, cp or None,
                          ctypes.addressof(tot), ctypes.addressof(nodes), stream or None)
    _check(rc, "dls_count")
    return int(tot.value), int(nodes.value)


def dls_count_async(n: int, depth: int, d_prefixes, d_counts, d_stats, symmetric: bool = False,
                    fixed_first_row: bool = True, stream: Optional[int] = None) -> None:
    """Enqueue the search on ``stream``; all tensors must be CUDA tensors."""
    k = _check_records(d_prefixes, n, "dls_count_async")
    _check_counts(d_counts, k, "dls_count_async", getattr(d_prefixes, "device", None))
    if d_stats is None or _dtype_name(d_stats) not in ("uint64", "int64") or int(np.prod(tuple(d_stats.shape))) < DLS_STATS_WORDS:
        raise ValueError("dls_count_async: stats must be %d uint64/int64 words" % DLS_STATS_WORDS)
    pp, k1 = _ptr(d_prefixes)
    cp, k2 = _ptr(d_counts)
    sp, k3 = _ptr(d_stats)
    rc = load().dls_count_async(n, int(symmetric), int(fixed_first_row), depth, pp or None,
                                int(d_prefixes.shape[0]), cp or None, sp, stream or None)
    _check(rc, "dls_count_async")


def dls_canonize(n: int, hourglasses, symmetric: bool = False, stream: Optional[int] = None) -> np.ndarray:
    """Alg. 5 on the GPU: class size of every canonic hourglass record, 0 otherwise."""
    recs = hourglasses
    k = int(recs.shape[0])
    out = np.zeros(max(k, 1), dtype=np.uint32)
    pp, keep = _ptr(recs)
    rc = load().dls_canonize(n, int(symmetric), pp or None, k, out.ctypes.data, stream or None)
    _check(rc, "dls_canonize")
    return out[:k]


def dls_count_sb(n: int, symmetric: bool = False, stream: Optional[int] = None) -> dict:
    """Alg. 6 on the GPU -> {count, hourglasses, classes, nodes} (first row fixed)."""
    vals = [ctypes.c_uint64(0) for _ in range(4)]
    rc = load().dls_count_sb(n, int(symmetric), *[ctypes.addressof(v) for v in vals], stream or None)
    _check(rc, "dls_count_sb")
    return {"count": vals[0].value, "hourglasses": vals[1].value, "classes": vals[2].value, "nodes": vals[3].value}


def dls_count_sb_range(n: int, begin: int, end: int, symmetric: bool = False, stream: Optional[int] = None) -> dict:
    """Alg. 6 over the diagonal workunits [begin, end) (end < 0: to the end)."""
    vals = [ctypes.c_uint64(0) for _ in range(4)]
    rc = load().dls_count_sb_range(n, int(symmetric), begin, end, *[ctypes.addressof(v) for v in vals], stream or None)
    _check(rc, "dls_count_sb_range")
    return {"count": vals[0].value, "hourglasses": vals[1].value, "classes": vals[2].value, "nodes": vals[3].value}


def dls_emit(n: int, depth: int, d_prefixes, d_out, symmetric: bool = False, fixed_first_row: bool = True,
             stream: Optional[int] = None) -> int:
    """Write every completion of the (CUDA) records into d_out (CUDA uint8, (cap, n, n));
    returns the number of completions."""
    k = _check_records(d_prefixes, n, "dls_emit")
    if d_out is not None:
        _check_records(d_out, n, "dls_emit (output)")
    pp, k1 = _ptr(d_prefixes)
    op, k2 = _ptr(d_out)
    cap = int(d_out.shape[0]) if d_out is not None else 0
    got = load().dls_emit(n, int(symmetric), int(fixed_first_row), depth, pp or None, int(d_prefixes.shape[0]),
                          op or None, cap, stream or None)
    _check(got, "dls_emit")
    return int(got)


def dls_count_cells(n: int, record: np.ndarray, cells, symmetric: bool = False, stream: Optional[int] = None):
    """Consistent assignments of `cells` below `record` -> (count, nodes)."""
    rec = np.ascontiguousarray(record, dtype=np.uint8).reshape(-1)
    cl = np.ascontiguousarray(np.asarray(list(cells), dtype=np.int32))
    tot = ctypes.c_uint64(0)
    nodes = ctypes.c_uint64(0)
    rc = load().dls_count_cells(n, int(symmetric), rec.ctypes.data, cl.ctypes.data if len(cl) else None, len(cl),
                                ctypes.addressof(tot), ctypes.addressof(nodes), stream or None)
    _check(rc, "dls_count_cells")
    return int(tot.value), int(nodes.value)


def dls_random_prefix(n: int, record: np.ndarray, cells, seed: int, symmetric: bool = False):
    """One Knuth random descent -> (record (n, n) uint8, weight)."""
    rec = np.ascontiguousarray(record, dtype=np.uint8).reshape(-1)
    cl = np.ascontiguousarray(np.asarray(list(cells), dtype=np.int32))
    out = np.empty(n * n, dtype=np.uint8)
    w = ctypes.c_double(0.0)
    rc = load().dls_random_prefix(n, int(symmetric), rec.ctypes.data, cl.ctypes.data if len(cl) else None, len(cl),
                                  ctypes.c_uint64(seed & (2 ** 64 - 1)), out.ctypes.data, ctypes.addressof(w))
    _check(rc, "dls_random_prefix")
    return out.reshape(n, n), float(w.value)


def dls_search_levels(n: int, depth: int, symmetric: bool = False, fixed_first_row: bool = True) -> int:
    """Plan cells the GPU search assigns below depth-`depth` records (the two-row
    closure level, or n_steps - depth); the reported nodes are their assignments."""
    out = ctypes.c_int32(0)
    rc = load().dls_search_levels(n, int(symmetric), int(fixed_first_row), depth, ctypes.addressof(out))
    _check(rc, "dls_search_levels")
    return int(out.value)


def dls_kernel_launches() -> int:
    return int(load().dls_kernel_launches())


def dls_scale_total(n: int, count_fixed: int, symmetric: bool = False):
    """-> (count_fixed * multiplier, multiplier): the full count from the first-row-fixed
    one (R3 for vertical symmetry).  128-bit product formed in the library."""
    out = (ctypes.c_uint64 * 2)()
    m = ctypes.c_uint64(0)
    _check(load().dls_scale_total(n, int(symmetric), ctypes.c_uint64(int(count_fixed)), ctypes.addressof(out),
                                  ctypes.addressof(m)), "dls_scale_total")
    return int(out[0]) | (int(out[1]) << 64), int(m.value)


def dls_mc_estimate(weights, counts, n_k: float):
    """Section 5.3 estimate from Knuth samples -> dict(knuth, knuth_se, ratio, mean_completions_weighted)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    if w.shape != c.shape or w.ndim != 1:
        raise ValueError("weights and counts must be 1-d arrays of equal length")
    out = np.zeros(4, dtype=np.float64)
    _check(load().dls_mc_estimate(w.ctypes.data, c.ctypes.data, int(w.shape[0]), float(n_k), out.ctypes.data),
           "dls_mc_estimate")
    return {"knuth": float(out[0]), "knuth_se": float(out[1]), "ratio": float(out[2]),
            "mean_completions_weighted": float(out[3])}
