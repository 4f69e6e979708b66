"""A/B of kernel options set through the environment on BASELINE configs 4/5
(seeded prefixes, dls_count with host refinement -- the public call), e.g.

    python scripts/ab_env.py --config dls9 --limit 128 --variants "DLS_CLOSE=1;DLS_CLOSE=0;DLS_LOOKAHEAD=51-60"

Every variant must give the same per-prefix counts (checked against the first).
Wall time around the synchronous call; one untimed warm-up call first.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1709_02599_b200 as D  # noqa: E402
import synth  # noqa: E402

KNOBS = ("DLS_CLOSE", "DLS_LOOKAHEAD", "DLS_CLOSE_FORCED", "DLS_MIN_DONATE", "DLS_CLOSE_MIN")


def run(n, vs, recs, env):
    for k in KNOBS:
        os.environ.pop(k, None)
    for kv in filter(None, env.split(",")):
        k, v = kv.split("=")
        os.environ[k.strip()] = v.strip()
    t = time.perf_counter()
    c, tot, nodes = D.count_prefixes(n, recs, vs)
    return c, {"variant": env or "default", "seconds": round(time.perf_counter() - t, 3), "squares": tot,
               "nodes": nodes, "squares_per_s": tot / (time.perf_counter() - t)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dls9", choices=["dls9", "vs10"])
    ap.add_argument("--limit", type=int, default=128)
    ap.add_argument("--variants", default="DLS_CLOSE=1;DLS_CLOSE=0")
    a = ap.parse_args()
    if a.config == "dls9":
        n, vs, recs = 9, False, synth.diagonal_prefixes(synth.SEED_DLS9, 9, synth.N_DLS9)[:a.limit]
    else:
        n, vs, recs = 10, True, synth.diagonal_prefixes(synth.SEED_VS10, 10, synth.N_VS10, vs=True)[:a.limit]
    run(n, vs, recs[:2], "")                      # warm-up: module load, pools
    base = None
    for env in a.variants.split(";"):
        c, r = run(n, vs, recs, env)
        if base is None:
            base = c
        r["counts_equal_first"] = bool((c == base).all())
        r.update(config=a.config, prefixes=len(recs))
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
