# final evidence run: full GPU tests, smoke, bench, ncu launch list of the bench command, ncu --set full captures, config timings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_full.log 2>&1; echo tests_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo ncul_rc=$?
timeout 300 python scripts/profile_kernel.py --n 8 --launches 3 > gpurun_out/prof_plain.log 2>&1; echo pk_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dls_search_kernel -s 1 -c 1 -o gpurun_out/r2_dls8_final python scripts/profile_kernel.py --n 8 --launches 2 > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dls_search_kernel -c 1 -o gpurun_out/r2_dls9_final python scripts/profile_kernel.py --n 9 --limit 8 --extra 6 --launches 1 > gpurun_out/ncu_full9.log 2>&1; echo ncu9_rc=$?
timeout 900 python scripts/time_configs.py > gpurun_out/time_configs.jsonl 2> gpurun_out/time_configs.err; echo tc_rc=$?
