cd $GRAFT_REPO_ROOT
O=gpurun_out/r2r
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gate_tc.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for v in base fw16 fw8; do
  MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate|assign" -c 9 --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_$v.csv 2>/dev/null
  MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_$v.so timeout 300 python bench.py --steps 30 --no-e2e --no-cpu-baseline > $O/b_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['phases_ms']['gate'], d['clocks']['sm_mhz'])"
done
