"""Per-prefix GPU counts of BASELINE configs 4/5: the indices of the smallest and
largest counts (the oracle then computes those prefixes: scripts/make_golden_r2.py
--indices-*), plus all counts for the record.

    python scripts/dump_minmax.py > gpurun_out/minmax.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1709_02599_b200 as D  # noqa: E402
import synth  # noqa: E402

out = {}
for tag, n, vs, seed, cnt in (("vs10", 10, True, synth.SEED_VS10, synth.N_VS10), ("dls9", 9, False, synth.SEED_DLS9, synth.N_DLS9)):
    recs = synth.diagonal_prefixes(seed, n, cnt, vs=vs)
    c, tot, nodes = D.count_prefixes(n, recs, vs)
    out[tag] = {"argmin": int(np.argmin(c)), "min": int(c.min()), "argmax": int(np.argmax(c)), "max": int(c.max()),
                "total": int(tot), "counts": [int(x) for x in c]}
print(json.dumps(out))
