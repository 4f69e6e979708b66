mkdir -p gpurun_out
P=$PWD/paper_1709_02599_b200
for i in 1 2; do
for v in "" _v_v1 _v_nouni; do
echo "variant libdls_b200$v" >> gpurun_out/ab_step2.log
DLS_LIB=$P/libdls_b200$v.so timeout 300 python scripts/profile_kernel.py --n 8 --launches 3 >> gpurun_out/ab_step2.log 2>&1
done
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_full.log 2>&1; echo tests_rc=$?
timeout 900 python scripts/time_configs.py > gpurun_out/time_configs.jsonl 2> gpurun_out/time_configs.err; echo tc_rc=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
