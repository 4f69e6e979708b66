"""Oracle counts for one seeded-random child of EVERY seeded prefix of BASELINE
configs 4 (VS10, 4096 prefixes) and 5 (DLS9, 1024 prefixes); calls only oracle/
and synth/.

    python scripts/make_golden_children.py [--workers 3]

For prefix i the child is a random descent of `extra` plan cells below it
(numpy default_rng(i); at every cell a uniform choice among the consistent
values the oracle lists; restart on a dead end), so every seeded prefix is
touched by an oracle comparison in tests/test_gpu_parity.py.  Per child:
completions, the oracle's full-tree nodes, and its nodes down to the two-row
level (the first level after which only two rows have empty cells, in the same
columns, off both diagonals -- DESIGN.md R15), computed here from that definition.
Output: tests/golden/children_{vs10,dls9}.txt.
"""
import argparse
import os
import sys
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
EXTRA = {"vs10": 8, "dls9": 12}


def two_row_level(n, vs, grid, order):
    """First l >= 1 (cells of `order` assigned) after which exactly two rows have
    empty cells, with the same empty columns and none on a diagonal; else len(order)."""
    empty = np.asarray(grid) == -1
    for l in range(0, len(order) + 1):
        if l:
            i, j = divmod(order[l - 1], n)
            empty[i, j] = False
            if vs:
                empty[i, n - 1 - j] = False
        rows = [i for i in range(n) if empty[i].any()]
        if len(rows) != 2 or (empty[rows[0]] != empty[rows[1]]).any():
            continue
        if any(empty[r, j] and (r == j or r + j == n - 1) for r in rows for j in range(n)):
            continue
        return l if l else len(order)
    return len(order)


def job(args):
    tag, n, vs, i, rec = args
    order = oracle.plan(n, vs)
    g = synth.to_int_grid(rec)
    d = sum(1 for c in order if g.reshape(-1)[c] != -1)
    rng = np.random.default_rng(i)
    for _ in range(10000):
        cur, ok = g.copy(), True
        for l in range(d, d + EXTRA[tag]):
            kids = oracle.prefixes(n, vs, cur, order[l:], 1, cap=64)
            if len(kids) == 0:
                ok = False
                break
            cur = kids[rng.integers(len(kids))]
        if ok:
            break
    rest = order[d + EXTRA[tag]:]
    c, lv = oracle.count_levels(n, vs, cur, rest)
    lc = two_row_level(n, vs, cur, rest)
    digits = "".join("." if v < 0 else str(int(v)) for v in cur.reshape(-1))
    return tag, i, digits, c, sum(lv), sum(lv[:lc])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=3)
    a = ap.parse_args()
    jobs = []
    for tag, n, vs, seed, cnt in (("vs10", 10, True, synth.SEED_VS10, synth.N_VS10),
                                  ("dls9", 9, False, synth.SEED_DLS9, synth.N_DLS9)):
        pre = synth.diagonal_prefixes(seed, n, cnt, vs=vs)
        jobs += [(tag, n, vs, i, pre[i]) for i in range(cnt)]
    with Pool(a.workers) as pool:
        res = pool.map(job, jobs, chunksize=16)
    for tag in EXTRA:
        rows = sorted(r for r in res if r[0] == tag)
        with open(os.path.join(GOLD, "children_%s.txt" % tag), "w") as f:
            f.write("# Written by scripts/make_golden_children.py (oracle + synth only): for every seeded\n"
                    "# prefix i, a default_rng(i) random descent of %d plan cells; the child record\n"
                    "# (row-major, '.' = empty), its completions, the oracle's full-tree nodes and its\n"
                    "# nodes down to the two-row level (DESIGN.md R15).\n"
                    "# index record count nodes nodes_two_row\n" % EXTRA[tag])
            for r in rows:
                f.write("%d %s %d %d %d\n" % r[1:])


if __name__ == "__main__":
    main()
