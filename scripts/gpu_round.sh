mkdir -p gpurun_out
P=$PWD/paper_1709_02599_b200
# correctness of the new paths first: column-only events (DLS_CLOSE_ROW8=1) and the lazy drain, product + checked build
DLS_CLOSE_ROW8=1 timeout 1200 python -m pytest tests -m gpu -x -q -k "closure or config1 or config2 or config3 or vs8 or small or smoke or few_workunits or pool_stress or ragged or checked or repeat or device_buffers or concurrent" > gpurun_out/tests_row8.log 2>&1; echo tests8_rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_full.log 2>&1; echo tests_rc=$?
for i in 1 2; do
echo "default (16-byte events, lazy drain)" >> gpurun_out/ab_row8.log
timeout 300 python scripts/profile_kernel.py --n 8 --launches 3 >> gpurun_out/ab_row8.log 2>&1
for t in 20 24 28; do
echo "ROW8 GROUP8=8 DLS_CLOSE_MIN=$t" >> gpurun_out/ab_row8.log
DLS_CLOSE_ROW8=1 DLS_CLOSE_MIN=$t timeout 300 python scripts/profile_kernel.py --n 8 --launches 3 >> gpurun_out/ab_row8.log 2>&1
done
echo "16-byte events, constants kept across the scheduling point (_v_nosp)" >> gpurun_out/ab_row8.log
DLS_LIB=$P/libdls_b200_v_nosp.so timeout 300 python scripts/profile_kernel.py --n 8 --launches 3 >> gpurun_out/ab_row8.log 2>&1
for v in _v_g6 _v_g12; do
echo "ROW8 $v DLS_CLOSE_MIN=24" >> gpurun_out/ab_row8.log
DLS_CLOSE_ROW8=1 DLS_LIB=$P/libdls_b200$v.so timeout 300 python scripts/profile_kernel.py --n 8 --launches 3 >> gpurun_out/ab_row8.log 2>&1
done
done
timeout 900 python scripts/time_configs.py > gpurun_out/time_configs_lazy.jsonl 2> gpurun_out/time_configs.err; echo tc_rc=$?
# resume the symmetry-broken DLS9 count (214 of 256 parts done in the previous call)
cp runs/sb9_r2_partial.jsonl gpurun_out/sb9_r2.jsonl
timeout 2400 python scripts/sb_full.py --n 9 --parts 256 --budget-s 2200 --out gpurun_out/sb9_r2.jsonl > gpurun_out/sb9_r2.log 2>&1; echo sb9_rc=$?
