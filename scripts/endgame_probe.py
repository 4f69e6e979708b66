"""End-game cost probe: one launch over all DLS8 workunits vs the same workunits
in 2 / 4 consecutive launches.  If the phase after the work queue runs dry were
as efficient as the rest, the sums would equal the single launch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1709_02599_b200 as D  # noqa: E402
from paper_1709_02599_b200 import _binding as B  # noqa: E402


def timed(n, d, dev, reps=3):
    st = torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        B.dls_count_async(n, d, dev, None, st, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best, int(st[0])


def main():
    n = 8
    d = D.default_split_depth(n)
    recs = torch.from_numpy(D.dls_split(n, d)).cuda()
    out = {"full": timed(n, d, recs)}
    for parts in (2, 4):
        m = recs.shape[0]
        res = [timed(n, d, recs[m * i // parts:m * (i + 1) // parts].contiguous()) for i in range(parts)]
        out["split%d" % parts] = (sum(r[0] for r in res), sum(r[1] for r in res), [round(r[0], 1) for r in res])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
