# long-run pins with the round-2 kernels: full VS10 and the symmetry-broken DLS8 / VS10 / DLS9
mkdir -p gpurun_out
python - > gpurun_out/sb_warm_r2.log 2>&1 <<'PY'
import time, json
import paper_1709_02599_b200 as D
for n, vs in ((8, False), (8, False), (8, False), (10, True), (10, True)):
    t = time.perf_counter(); r = D.dls_count_sb(n, vs); dt = time.perf_counter() - t
    print(json.dumps({"n": n, "vs": vs, "seconds": round(dt, 3), **{k: (int(v) if hasattr(v, "__int__") else v) for k, v in r.items()}}), flush=True)
PY
echo sb_rc=$?
rm -f gpurun_out/vs10_full_r2.jsonl
timeout 3000 python scripts/vs10_full.py --chunks 16 --out gpurun_out/vs10_full_r2.jsonl > gpurun_out/vs10_full_r2.log 2>&1; echo vs10_rc=$?
rm -f gpurun_out/sb9_r2.jsonl
timeout 5400 python scripts/sb_full.py --n 9 --parts 256 --budget-s 5000 --out gpurun_out/sb9_r2.jsonl > gpurun_out/sb9_r2.log 2>&1; echo sb9_rc=$?
