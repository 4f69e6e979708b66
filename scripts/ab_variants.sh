for r in 1 2; do
for v in ${VARIANTS:-"" _v10 _v01 _v11}; do
  DLS_LIB=$PWD/paper_1709_02599_b200/libdls_b200$v.so timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
