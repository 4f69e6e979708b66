mkdir -p gpurun_out
P=$PWD/paper_1709_02599_b200
timeout 900 python scripts/ab_env.py --config dls9 --limit 64 --variants "DLS_CLOSE=1;DLS_CLOSE=0" > gpurun_out/ab_dls9_uni.log 2>&1; echo ab9_rc=$?
DLS_LIB=$P/libdls_b200_v_nouni.so timeout 900 python scripts/ab_env.py --config dls9 --limit 64 --variants "DLS_CLOSE=1;DLS_CLOSE=0" > gpurun_out/ab_dls9_nouni.log 2>&1
timeout 900 python scripts/ab_env.py --config vs10 --limit 256 --variants "DLS_CLOSE=1;DLS_CLOSE=0" > gpurun_out/ab_vs10_uni.log 2>&1; echo ab10_rc=$?
DLS_LIB=$P/libdls_b200_v_nouni.so timeout 900 python scripts/ab_env.py --config vs10 --limit 256 --variants "DLS_CLOSE=1" > gpurun_out/ab_vs10_nouni.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_full.log 2>&1; echo tests_rc=$?
