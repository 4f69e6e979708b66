"""Round-2 golden extension: oracle counts of a stratified sample of the BASELINE
config 4 / 5 seeded prefixes (calls only oracle/ and synth/).

    python scripts/make_golden_r2.py [--workers 5]

Strata: the seeded prefix list is cut into equal-width index strata and one index
is drawn per stratum from numpy's default_rng(2026) (indices already in the
round-1 files are skipped).  Each finished count is appended (and flushed) to
tests/golden/{dls9,vs10}_prefix_counts_r2.txt, so an interrupted run keeps what
it has.  Longest jobs (DLS9, about 2 CPU-hours each) are scheduled first.
"""
import argparse
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
R1 = {"vs10": [0, 1, 2, 3, 1000, 2000, 3000, 4095], "dls9": [0, 1, 2, 3, 256, 512, 768, 1023]}


def strata(total, k, skip, seed=2026):
    rng = np.random.default_rng(seed)
    edges = np.linspace(0, total, k + 1).astype(int)
    out = []
    for a, b in zip(edges[:-1], edges[1:]):
        cand = [i for i in range(a, b) if i not in skip]
        out.append(int(rng.choice(cand)))
    return out


def job(args):
    tag, n, vs, idx, rec = args
    t = time.time()
    c, nodes = oracle.count(n, vs, synth.to_int_grid(rec))
    return tag, idx, c, nodes, time.time() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=5)
    ap.add_argument("--dls9", type=int, default=10)
    ap.add_argument("--vs10", type=int, default=24)
    ap.add_argument("--indices-dls9", default="", help="comma-separated seeded-prefix indices to add (e.g. the GPU's min / max counts)")
    ap.add_argument("--indices-vs10", default="")
    a = ap.parse_args()
    extra = {"dls9": [int(x) for x in a.indices_dls9.split(",") if x], "vs10": [int(x) for x in a.indices_vs10.split(",") if x]}
    jobs = []
    pre9 = synth.diagonal_prefixes(synth.SEED_DLS9, 9, synth.N_DLS9)
    pre10 = synth.diagonal_prefixes(synth.SEED_VS10, 10, synth.N_VS10, vs=True)
    for tag, n, vs, pre, k, seed in (("dls9", 9, False, pre9, a.dls9, synth.SEED_DLS9),
                                     ("vs10", 10, True, pre10, a.vs10, synth.SEED_VS10)):
        path = os.path.join(GOLD, "%s_prefix_counts_r2.txt" % tag)
        done = set()
        if os.path.exists(path):
            done = {int(l.split()[0]) for l in open(path) if l.strip() and not l.startswith("#")}
        else:
            with open(path, "w") as f:
                f.write("# Written by scripts/make_golden_r2.py: oracle.count on synth.diagonal_prefixes("
                        "seed=%d, n=%d, vs=%s) records,\n# one index per equal-width stratum "
                        "(default_rng(2026)).\n# index count nodes oracle_seconds\n" % (seed, n, vs))
        for i in (strata(len(pre), k, set(R1[tag])) if k > 0 else []) + extra[tag]:
            if i not in done and i not in R1[tag]:
                jobs.append((tag, n, vs, i, pre[i]))
    with Pool(a.workers) as pool:
        for tag, idx, c, nodes, sec in pool.imap_unordered(job, jobs, chunksize=1):
            with open(os.path.join(GOLD, "%s_prefix_counts_r2.txt" % tag), "a") as f:
                f.write("%d %d %d %.1f\n" % (idx, c, nodes, sec))
            print(tag, idx, c, sec, flush=True)


if __name__ == "__main__":
    main()
