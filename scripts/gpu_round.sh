# second GPU call of round 2: smoke, ncu launch list + full capture of the bench kernel, DLS9 A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python scripts/ab_env.py --config dls9 --limit 96 --variants "DLS_CLOSE=1;DLS_CLOSE=0;DLS_LOOKAHEAD=51-60;DLS_CLOSE=0,DLS_LOOKAHEAD=51-60" > gpurun_out/ab_dls9.log 2>&1; echo ab_rc=$?
timeout 600 python scripts/profile_kernel.py --n 8 --launches 1 > gpurun_out/prof_plain.log 2>&1; echo pk_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dls_search_kernel -c 1 -o gpurun_out/r2_dls8_close python scripts/profile_kernel.py --n 8 --launches 1 > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncul_rc=$?
