mkdir -p gpurun_out
P=$PWD/paper_1709_02599_b200
for i in 1 2; do
for v in "" _v_sa _v_full _v_full12 _v_safull; do
echo "variant libdls_b200$v" >> gpurun_out/ab_step5.log
DLS_LIB=$P/libdls_b200$v.so timeout 300 python scripts/profile_kernel.py --n 8 --launches 3 >> gpurun_out/ab_step5.log 2>&1
done
done
for v in "" _v_sa; do
echo "variant libdls_b200$v dls9" >> gpurun_out/ab_step5.log
DLS_LIB=$P/libdls_b200$v.so timeout 600 python scripts/ab_env.py --config dls9 --limit 64 --variants "DLS_CLOSE=1" >> gpurun_out/ab_step5.log 2>&1
echo "variant libdls_b200$v vs10" >> gpurun_out/ab_step5.log
DLS_LIB=$P/libdls_b200$v.so timeout 600 python scripts/ab_env.py --config vs10 --limit 256 --variants "DLS_CLOSE=1" >> gpurun_out/ab_step5.log 2>&1
done
timeout 600 python scripts/dump_minmax.py > gpurun_out/minmax.json 2> gpurun_out/minmax.err; echo minmax_rc=$?
