"""Small runs of every kernel (search, device pool, emit, hourglass + canonise,
symmetry breaking, cells).  compute-sanitizer is closed on the GPU pool; run this
with DLS_LIB=paper_1709_02599_b200/libdls_b200_checked.so to exercise the
kernels' own invariants (DLS_CHECK) instead."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1709_02599_b200 as D  # noqa: E402
from paper_1709_02599_b200 import _binding as B  # noqa: E402

out = {}
out["dls6_free"] = D.count_squares(6, fixed_first_row=False)["count"]          # dls_count + refinement
out["vs8"] = D.count_squares(8, True)["count"]
d = D.default_split_depth(7)
recs = torch.from_numpy(D.dls_split(7, d)[:3]).cuda()                          # device pool spreading
st = torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device="cuda")
D.dls_count_async(7, d, recs, None, st, stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
out["dls7_3wu"] = int(st[0])
buf = torch.zeros((200, 5, 5), dtype=torch.uint8, device="cuda")
r5 = torch.from_numpy(D.dls_split(5, D.default_split_depth(5))).cuda()
out["emit5"] = D.dls_emit(5, D.default_split_depth(5), r5, buf)                # emit kernel
out["sb7"] = D.dls_count_sb(7)["count"]                                        # hourglass + canonize
out["sb6vs"] = D.dls_count_sb(6, True)["count"]
g = np.full((6, 6), 255, np.uint8)
g[0] = np.arange(6)
out["cells6"] = D.dls_count_cells(6, g, list(range(6, 18)))[0]
print(out)
