"""Time the phases of one end-to-end N=8 enumeration through the public API."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1709_02599_b200 as D  # noqa: E402
from paper_1709_02599_b200 import _binding as B  # noqa: E402


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


def main():
    n, d = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 14
    D.count_squares(n, depth=d)          # warm-up (context, module load)
    for rep in range(int(os.environ.get("REPS", "3"))):
        t0 = t()
        lib = B.load()
        total = lib.dls_split(n, 0, 1, d, None, 0)
        t1 = t()
        recs = np.empty((total, n, n), np.uint8)
        lib.dls_split(n, 0, 1, d, recs.ctypes.data, total)
        t2 = t()
        tot, nodes = D.dls_count(n, d, recs)
        t3 = t()
        pinned = torch.empty((total, n, n), dtype=torch.uint8).pin_memory()
        t4 = t()
        lib.dls_split(n, 0, 1, d, pinned.data_ptr(), total)
        t5 = t()
        tot2, _ = D.dls_count(n, d, pinned)
        t6 = t()
        dev = torch.from_numpy(recs).cuda()
        t7 = t()
        tot3, _ = D.dls_count(n, d, dev)
        t8 = t()
        print("rep %d: split-count %.1f ms, split-fill %.1f ms, count(pageable) %.1f ms, pin-alloc %.1f ms, "
              "split-into-pinned %.1f ms, count(pinned) %.1f ms, H2D torch %.1f ms, count(device) %.1f ms  [%d %d %d]"
              % (rep, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3), 1e3 * (t5 - t4),
                 1e3 * (t6 - t5), 1e3 * (t7 - t6), 1e3 * (t8 - t7), tot, tot2, tot3))


if __name__ == "__main__":
    main()
