"""Time BASELINE configs 4/5 through the public API (dls_count with host refinement)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1709_02599_b200 as D  # noqa: E402
import synth  # noqa: E402


def run(n, vs, seed, count, limit):
    recs = synth.diagonal_prefixes(seed, n, count, vs=vs)[:limit]
    torch.cuda.synchronize()
    t = time.perf_counter()
    c, tot, nodes = D.count_prefixes(n, recs, vs)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return {"n": n, "vs": vs, "prefixes": len(recs), "seconds": dt, "squares": tot, "nodes": nodes,
            "squares_per_s": tot / dt, "nodes_per_s": nodes / dt, "first_counts": [int(x) for x in c[:4]]}


if __name__ == "__main__":
    which = sys.argv[1:] or ["vs10", "dls9"]
    if "vs10" in which:
        print(json.dumps(run(10, True, synth.SEED_VS10, synth.N_VS10, int(os.environ.get("LIMIT", "4096")))), flush=True)
    if "dls9" in which:
        print(json.dumps(run(9, False, synth.SEED_DLS9, synth.N_DLS9, int(os.environ.get("LIMIT", "1024")))), flush=True)
