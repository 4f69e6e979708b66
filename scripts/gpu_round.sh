mkdir -p gpurun_out
P=$PWD/paper_1709_02599_b200
for i in 1 2; do
for v in "" _v_rd8; do
echo "variant libdls_b200$v" >> gpurun_out/ab_step4.log
DLS_LIB=$P/libdls_b200$v.so timeout 300 python scripts/profile_kernel.py --n 8 --launches 3 >> gpurun_out/ab_step4.log 2>&1
done
done
bash scripts/gpu_long.sh
