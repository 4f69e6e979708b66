"""Command line over the C ABI (every computation runs in libdls_b200.so).

    python -m paper_1709_02599_b200 plan  --n 9                  # Section 2.3 order (Fig. 1 layout)
    python -m paper_1709_02599_b200 split --n 9 --depth 10       # number of workunits
    python -m paper_1709_02599_b200 count --n 8 [--vs] [--free]  # exhaustive GPU count
    python -m paper_1709_02599_b200 count --n 10 --vs --sb       # with symmetry breaking (Alg. 6)
    python -m paper_1709_02599_b200 cells --n 10 --k 32          # N_n^k of Section 5.3
    python -m paper_1709_02599_b200 estimate --n 10 --k 32 --samples 16
"""
import argparse
import json
import math
import sys
import time

import numpy as np

from . import _binding as B
from .api import count_squares


def cmd_plan(a):
    cells, forced, dd = B.dls_plan(a.n, a.vs, not a.free)
    grid = np.zeros((a.n, a.n), dtype=int)
    for s, c in enumerate(cells):
        grid[c // a.n, c % a.n] = s + 1
    for i in range(a.n):
        print(" ".join("%3s" % ("-" if grid[i, j] == 0 else grid[i, j]) for j in range(a.n)))
    print("diagonal depth:", dd, " forced steps:", [s + 1 for s in range(len(cells)) if forced[s]])


def cmd_split(a):
    print(B.load().dls_split(a.n, int(a.vs), int(not a.free), a.depth, None, 0))


def cmd_count(a):
    t = time.perf_counter()
    if a.sb:
        r = B.dls_count_sb(a.n, a.vs)
    else:
        r = count_squares(a.n, a.vs, not a.free)
    r["seconds"] = time.perf_counter() - t
    if not a.free:
        r["total_all_first_rows"] = B.dls_scale_total(a.n, r["count"], a.vs)[0]
    print(json.dumps(r))


def cmd_cells(a):
    rec = np.full((a.n, a.n), 255, np.uint8)
    rec[0, :] = np.arange(a.n)
    t = time.perf_counter()
    c, nodes = B.dls_count_cells(a.n, rec, list(range(a.n, a.k)), a.vs)
    print(json.dumps({"n": a.n, "k": a.k, "count": c, "nodes": nodes, "seconds": time.perf_counter() - t}))


def cmd_estimate(a):
    rec = np.full((a.n, a.n), 255, np.uint8)
    rec[0, :] = np.arange(a.n)
    cells = list(range(a.n, a.k))
    ws, cs = [], []
    for s in range(a.samples):
        pre, w = B.dls_random_prefix(a.n, rec, cells, a.seed * 1000003 + s, a.vs)
        c = 0
        if w > 0:
            rest = [i for i in range(a.n * a.n) if pre.reshape(-1)[i] == 255 and (not a.vs or 2 * (i % a.n) <= a.n - 1)]
            c, _ = B.dls_count_cells(a.n, pre, rest, a.vs)
        ws.append(w)
        cs.append(c)
    est = B.dls_mc_estimate(ws, cs, 0.0)
    print(json.dumps({"n": a.n, "k": a.k, "samples": a.samples, "estimate": est["knuth"],
                      "stderr": None if a.samples < 2 else est["knuth_se"]}))


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1709_02599_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name, fn in (("plan", cmd_plan), ("split", cmd_split), ("count", cmd_count), ("cells", cmd_cells),
                     ("estimate", cmd_estimate)):
        p = sub.add_parser(name)
        p.add_argument("--n", type=int, required=True)
        p.add_argument("--vs", action="store_true", help="vertically symmetric (P:521)")
        p.add_argument("--free", action="store_true", help="do not fix row 0 (P:112)")
        p.set_defaults(fn=fn)
        if name == "split":
            p.add_argument("--depth", type=int, required=True)
        if name == "count":
            p.add_argument("--sb", action="store_true", help="symmetry breaking (Alg. 6)")
        if name in ("cells", "estimate"):
            p.add_argument("--k", type=int, required=True)
        if name == "estimate":
            p.add_argument("--samples", type=int, default=16)
            p.add_argument("--seed", type=int, default=1)
    a = ap.parse_args(argv)
    try:
        a.fn(a)
    except B.DlsError as e:
        print("error: %s" % e, file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
