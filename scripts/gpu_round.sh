mkdir -p gpurun_out
P=$PWD/paper_1709_02599_b200
for i in 1 2; do
for v in "" _v_v3 _v_v4 _v_v34 _v_v34f _v_v3f; do
echo "variant libdls_b200$v" >> gpurun_out/ab_step3.log
DLS_LIB=$P/libdls_b200$v.so timeout 300 python scripts/profile_kernel.py --n 8 --launches 3 >> gpurun_out/ab_step3.log 2>&1
done
done
for v in "" _v_v3 _v_v3f; do
echo "variant libdls_b200$v dls9" >> gpurun_out/ab_step3.log
DLS_LIB=$P/libdls_b200$v.so timeout 600 python scripts/ab_env.py --config dls9 --limit 64 --variants "DLS_CLOSE=1" >> gpurun_out/ab_step3.log 2>&1
echo "variant libdls_b200$v vs10" >> gpurun_out/ab_step3.log
DLS_LIB=$P/libdls_b200$v.so timeout 600 python scripts/ab_env.py --config vs10 --limit 256 --variants "DLS_CLOSE=1" >> gpurun_out/ab_step3.log 2>&1
done
