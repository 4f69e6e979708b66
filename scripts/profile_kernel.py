"""Launch the search kernel a few times on one workload (for ncu / quick timing).

    python scripts/profile_kernel.py [--n 8] [--vs] [--depth D] [--launches 2] [--limit K] [--extra E]

N <= 8: all workunits of the first-row-fixed problem at depth D (default: diagonals).
N >= 9: the seeded diagonal prefixes of BASELINE configs 4/5 (first --limit of them).
--extra E refines the records E plan cells deeper on the host (dls_refine).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1709_02599_b200 as D  # noqa: E402
from paper_1709_02599_b200 import _binding as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--vs", action="store_true")
    ap.add_argument("--depth", type=int, default=None)
    ap.add_argument("--launches", type=int, default=2)
    ap.add_argument("--limit", type=int, default=0)
    ap.add_argument("--extra", type=int, default=0)
    a = ap.parse_args()
    d = D.default_split_depth(a.n, a.vs) if a.depth is None else a.depth
    if a.n >= 9 and a.depth is None:
        import synth
        recs = synth.diagonal_prefixes(synth.SEED_VS10 if a.vs else synth.SEED_DLS9, a.n, a.limit or 64, vs=a.vs)
    else:
        recs = D.dls_split(a.n, d, a.vs)
        if a.limit:
            recs = recs[:a.limit]
    if a.extra:
        recs, _ = D.dls_refine(a.n, d, recs, d + a.extra, a.vs)
        d += a.extra
    dev = torch.from_numpy(recs).cuda()
    stats = torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    out = []
    for i in range(a.launches):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        B.dls_count_async(a.n, d, dev, None, stats, a.vs, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        st = stats.cpu().tolist()
        ms = e0.elapsed_time(e1)
        out.append({"launch": i, "ms": ms, "count": st[0], "nodes": st[1], "err": st[2],
                    "donations": st[4], "pool": st[7], "lane_util": st[5] / max(st[6], 1),
                    "squares_per_s": st[0] / ms * 1e3, "nodes_per_s": st[1] / ms * 1e3})
    print(json.dumps({"n": a.n, "vs": a.vs, "depth": d, "n_prefix": int(recs.shape[0]),
                      "donate": os.environ.get("DLS_DONATE", "1"), "launches": out}), flush=True)


if __name__ == "__main__":
    main()
