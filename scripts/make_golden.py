"""Write oracle-computed expected values into tests/golden/ (calls only oracle/ and synth/).

    python scripts/make_golden.py [--workers 7]

Per-prefix completion counts of a fixed subset of BASELINE config 4 (VS, N=10,
seed synth.SEED_VS10) and config 5 (DLS, N=9, seed synth.SEED_DLS9) prefixes, and
the number of depth-10 workunits for N=9.  Each oracle count of a full
diagonal prefix takes minutes, hence stored rather than recomputed in tests.
"""
import argparse
import os
import sys
import time
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
VS10_IDX = [0, 1, 2, 3, 1000, 2000, 3000, 4095]
DLS9_IDX = [0, 1, 2, 3, 256, 512, 768, 1023]


def job(args):
    n, vs, idx, rec = args
    g = synth.to_int_grid(rec)
    t = time.time()
    c, nodes = oracle.count(n, vs, g)
    return n, vs, idx, c, nodes, time.time() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=7)
    ap.add_argument("--which", default="vs10,dls9,k10")
    a = ap.parse_args()
    jobs = []
    if "vs10" in a.which:
        pre = synth.diagonal_prefixes(synth.SEED_VS10, 10, max(VS10_IDX) + 1, vs=True)
        jobs += [(10, True, i, pre[i]) for i in VS10_IDX]
    if "dls9" in a.which:
        pre = synth.diagonal_prefixes(synth.SEED_DLS9, 9, max(DLS9_IDX) + 1)
        jobs += [(9, False, i, pre[i]) for i in DLS9_IDX]
    if "k10" in a.which:
        g = oracle.first_row_grid(9)
        k10 = oracle.count_prefixes(9, False, g, oracle.plan(9), 10)
        with open(os.path.join(GOLD, "dls9_k10_workunits.txt"), "w") as f:
            f.write("# Written by scripts/make_golden.py with oracle.count_prefixes (oracle only).\n"
                    "# Consistent assignments of the first 10 Fig. 1 cells for N=9, first row fixed.\n"
                    "# P:481 prints 1 225 884; see DESIGN.md reading R8.\n%d\n" % k10)
    with Pool(a.workers) as pool:
        res = pool.map(job, jobs, chunksize=1)
    for tag, n, vs in (("vs10", 10, True), ("dls9", 9, False)):
        rows = [r for r in res if r[0] == n and r[1] == vs]
        if not rows:
            continue
        with open(os.path.join(GOLD, "%s_prefix_counts.txt" % tag), "w") as f:
            f.write("# Written by scripts/make_golden.py: oracle.count on synth.diagonal_prefixes("
                    "seed=%d, n=%d, vs=%s) records.\n# index count nodes oracle_seconds\n"
                    % (synth.SEED_VS10 if vs else synth.SEED_DLS9, n, vs))
            for r in sorted(rows, key=lambda r: r[2]):
                f.write("%d %d %d %.1f\n" % (r[2], r[3], r[4], r[5]))


if __name__ == "__main__":
    main()
