"""paper_1709_02599_b200 -- B200-native (sm_100a) enumeration of diagonal Latin squares.

The data-parallel hot path of arXiv:1709.02599 (Kochemazov, Vatutin, Zaikin):
Section 2.3 cell order -> prefix split -> bit-arithmetic DFS (Alg. 4,
P:235-258) on every lane of a persistent CUDA kernel.  The C ABI is
include/dls_b200.h; this package is its thin binding plus convenience wrappers.
"""
from ._binding import (DLS_EMPTY, DLS_MAX_ORDER, DLS_STATS_WORDS, DlsError, dls_canonize, dls_count,  # noqa: F401
                       dls_count_async, dls_count_cells, dls_count_sb, dls_count_sb_range, dls_emit, dls_random_prefix,
                       dls_kernel_launches, dls_mc_estimate, dls_plan, dls_refine, dls_scale_total, dls_search_levels,
                       dls_split,
                       dls_version,
                       lib_path, load)
from .api import count_squares, default_split_depth, count_prefixes  # noqa: F401
