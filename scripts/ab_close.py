"""A/B of the two-row tail closure (DLS_CLOSE=1 default vs 0): same records,
counts must agree; prints kernel times (CUDA events, dls_count_async).

    python scripts/ab_close.py [--launches 3] [--cases dls8,vs8,dls7,vs10,dls9,dls10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1709_02599_b200 as D  # noqa: E402
import synth  # noqa: E402
from paper_1709_02599_b200 import _binding as B  # noqa: E402


def records(case):
    if case in ("dls8", "vs8", "dls7", "vs6"):
        n, vs = int(case[-1]), case.startswith("vs")
        d = D.default_split_depth(n, vs)
        return n, vs, d, D.dls_split(n, d, vs)
    if case == "vs10":
        n, vs = 10, True
        recs = synth.diagonal_prefixes(synth.SEED_VS10, 10, 64, vs=True)
    elif case == "dls9":
        n, vs = 9, False
        recs = synth.diagonal_prefixes(synth.SEED_DLS9, 9, 16)
    else:   # dls10: deep records (first 4 rows)
        n, vs = 10, False
        d = D.default_split_depth(n, vs)
        base = synth.diagonal_prefixes(7, 10, 1)
        recs, _ = D.dls_refine(n, d, base, d + 20, vs)
        return n, vs, d + 20, recs[:200000]
    d = D.default_split_depth(n, vs)
    recs, _ = D.dls_refine(n, d, recs, d + 4, vs)
    return n, vs, d + 4, recs


def run(n, vs, d, dev, launches):
    stats = torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device="cuda")
    counts = torch.zeros(dev.shape[0], dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    out = []
    for i in range(launches):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        B.dls_count_async(n, d, dev, counts, stats, vs, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        st = stats.cpu().tolist()
        out.append((e0.elapsed_time(e1), st[0], st[1], st[2]))
    return out, counts.cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--cases", default="dls7,vs8,dls8,vs10,dls9")
    a = ap.parse_args()
    for case in a.cases.split(","):
        n, vs, d, recs = records(case)
        dev = torch.from_numpy(np.ascontiguousarray(recs)).cuda()
        res = {}
        for close in ("1", "0"):
            os.environ["DLS_CLOSE"] = close
            res[close] = run(n, vs, d, dev, a.launches)
        os.environ["DLS_CLOSE"] = "1"
        (r1, c1), (r0, c0) = res["1"], res["0"]
        print(json.dumps({"case": case, "n_prefix": int(recs.shape[0]), "depth": d,
                          "counts_equal": bool((c1 == c0).all()), "total": [r1[-1][1], r0[-1][1]],
                          "nodes": [r1[-1][2], r0[-1][2]], "err": [r1[-1][3], r0[-1][3]],
                          "ms_close": [round(x[0], 2) for x in r1], "ms_plain": [round(x[0], 2) for x in r0]}),
              flush=True)


if __name__ == "__main__":
    main()
