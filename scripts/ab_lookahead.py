"""A/B of the lookahead of Section 2.4.2 on BASELINE config 5 (DLS9,
seeded prefixes): DLS_LOOKAHEAD unset vs the paper's loops 51-60 (and a wider
range); per-prefix counts must agree exactly.  dls_count with host refinement,
wall time around the call (synchronous).

    python scripts/ab_lookahead.py [--limit 256] [--ranges 51-60,41-60]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1709_02599_b200 as D  # noqa: E402
import synth  # noqa: E402


def run(recs, la):
    if la:
        os.environ["DLS_LOOKAHEAD"] = la
    else:
        os.environ.pop("DLS_LOOKAHEAD", None)
    t = time.perf_counter()
    c, tot, nodes = D.count_prefixes(9, recs)
    dt = time.perf_counter() - t
    return c, {"lookahead": la or "off", "seconds": dt, "squares": tot, "nodes": nodes,
               "squares_per_s": tot / dt, "nodes_per_s": nodes / dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--limit", type=int, default=256)
    ap.add_argument("--ranges", default="51-60,41-60")
    a = ap.parse_args()
    recs = synth.diagonal_prefixes(synth.SEED_DLS9, 9, synth.N_DLS9)[:a.limit]
    run(recs[:4], None)                                   # warm-up (module load)
    base_c, base = run(recs, None)
    print(json.dumps(dict(base, prefixes=len(recs))), flush=True)
    for la in a.ranges.split(","):
        c, r = run(recs, la)
        r["counts_equal"] = bool((c == base_c).all())
        r["speedup"] = base["seconds"] / r["seconds"]
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
