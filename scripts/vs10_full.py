"""Full count of vertically symmetric DLS of order 10 with the first row fixed
(82 731 715 264 512) on one B200, in resumable chunks.

    python scripts/vs10_full.py [--chunks 16] [--out gpurun_out/vs10_full.jsonl]

Every one of the 81 088 diagonal workunits (first row + both diagonals, mirror
consistent) is counted by dls_count; one JSON line per chunk is appended to the
output (chunk index, workunits, squares, nodes, seconds) so an interrupted run
can be resumed.  The last line holds the total.
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

PAPER_VS10 = 82731715264512   # P:524 (first row fixed, reading R2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=16)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "vs10_full.jsonl"))
    a = ap.parse_args()
    n, vs = 10, True
    d = D.default_split_depth(n, vs)
    recs = D.dls_split(n, d, vs)
    done = {}
    if os.path.exists(a.out):
        for line in open(a.out):
            r = json.loads(line)
            if "chunk" in r:
                done[r["chunk"]] = r
    bounds = np.linspace(0, len(recs), a.chunks + 1).astype(int)
    for k in range(a.chunks):
        if k in done:
            continue
        part = recs[bounds[k]:bounds[k + 1]]
        t = time.perf_counter()
        tot, nodes = D.dls_count(n, d, part, vs)
        dt = time.perf_counter() - t
        r = {"chunk": k, "workunits": int(len(part)), "squares": tot, "nodes": nodes, "seconds": dt}
        done[k] = r
        with open(a.out, "a") as f:
            f.write(json.dumps(r) + "\n")
        print(json.dumps(r), flush=True)
    total = sum(r["squares"] for r in done.values())
    secs = sum(r["seconds"] for r in done.values())
    nodes = sum(r["nodes"] for r in done.values())
    summary = {"total": total, "paper": PAPER_VS10, "match": total == PAPER_VS10, "workunits": int(len(recs)),
               "seconds": secs, "nodes": nodes, "squares_per_s": total / secs, "nodes_per_s": nodes / secs}
    with open(a.out, "a") as f:
        f.write(json.dumps(summary) + "\n")
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
