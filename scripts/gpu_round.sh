# last checks: full GPU tests with the complete round-2 golden files, VS10 ncu capture, then a longer Monte Carlo run
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_full.log 2>&1; echo tests_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dls_search_kernel -c 1 -o gpurun_out/r2_vs10_final python scripts/profile_kernel.py --n 10 --vs --limit 4 --extra 3 --launches 1 > gpurun_out/ncu_full10.log 2>&1; echo ncu10_rc=$?
timeout 3000 python scripts/mc_estimate.py --n 10 --k 32 --samples 448 --seed 5 > gpurun_out/mc_dls10_448.json 2> gpurun_out/mc.err; echo mc_rc=$?
