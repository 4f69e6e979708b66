"""Symmetry-broken full count (Alg. 6) in resumable parts.

    python scripts/sb_full.py --n 9 [--vs] [--parts 32] [--budget-s 3000] [--out gpurun_out/sb9.jsonl]

The diagonal workunits are cut into --parts ranges; each range goes through
dls_count_sb_range (GPU hourglass enumeration + canonisation + search of the
canonic designs) and one JSON line is appended per range.  Ranges already in the
output file are skipped, so the run can be spread over several calls.  When all
ranges are done a summary line is appended (total vs the paper's count).
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

PAPER = {(8, False): 7447587840, (9, False): 5056994653507584, (10, True): 82731715264512}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=9)
    ap.add_argument("--vs", action="store_true")
    ap.add_argument("--parts", type=int, default=32)
    ap.add_argument("--budget-s", type=float, default=1e9)
    ap.add_argument("--out", default=None)
    ap.add_argument("--resume-from", default=None, help="extra JSONL file of finished parts (read only)")
    a = ap.parse_args()
    out = a.out or os.path.join(ROOT, "gpurun_out", "sb%d%s.jsonl" % (a.n, "vs" if a.vs else ""))
    d = D.default_split_depth(a.n, a.vs)
    total_wu = D.load().dls_split(a.n, int(a.vs), 1, d, None, 0)
    bounds = np.linspace(0, total_wu, a.parts + 1).astype(np.int64)
    done = {}
    for path in (a.resume_from, out):
        if path and os.path.exists(path):
            for line in open(path):
                r = json.loads(line)
                if "part" in r and r.get("parts") == a.parts:
                    done[r["part"]] = r
    t_start = time.perf_counter()
    for k in range(a.parts):
        if k in done:
            continue
        if time.perf_counter() - t_start > a.budget_s:
            break
        t = time.perf_counter()
        r = D.dls_count_sb_range(a.n, int(bounds[k]), int(bounds[k + 1]), a.vs)
        r.update({"part": k, "parts": a.parts, "begin": int(bounds[k]), "end": int(bounds[k + 1]),
                  "seconds": time.perf_counter() - t})
        done[k] = r
        with open(out, "a") as f:
            f.write(json.dumps(r) + "\n")
        print(json.dumps(r), flush=True)
    if len(done) == a.parts:
        tot = sum(r["count"] for r in done.values())
        summ = {"n": a.n, "vs": a.vs, "total": tot, "paper": PAPER.get((a.n, a.vs)),
                "match": tot == PAPER.get((a.n, a.vs)),
                "hourglasses": sum(r["hourglasses"] for r in done.values()),
                "classes": sum(r["classes"] for r in done.values()),
                "nodes": sum(r["nodes"] for r in done.values()),
                "seconds": sum(r["seconds"] for r in done.values())}
        with open(out, "a") as f:
            f.write(json.dumps(summ) + "\n")
        print(json.dumps(summ), flush=True)


if __name__ == "__main__":
    main()
