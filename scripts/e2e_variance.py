"""Back-to-back dls_count calls with pinned host records (the bench's e2e step),
with per-call wall time; run with DLS_TIMING=1 for the per-launch timeline."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1709_02599_b200 as D  # noqa: E402
from paper_1709_02599_b200 import _binding as B  # noqa: E402

n, d = 8, 14
lib = B.load()
total = lib.dls_split(n, 0, 1, d, None, 0)
pin = torch.empty((total, n, n), dtype=torch.uint8).pin_memory()
out = []
for i in range(int(os.environ.get("REPS", "12"))):
    t = time.perf_counter()
    lib.dls_split(n, 0, 1, d, pin.data_ptr(), total)
    tot, _ = D.dls_count(n, d, pin)
    out.append(round((time.perf_counter() - t) * 1e3, 1))
    assert tot == 7447587840
print(json.dumps({"ms": out}))
