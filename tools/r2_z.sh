cd $GRAFT_REPO_ROOT
O=gpurun_out/r2z
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_layer.py tests/test_gpu_ops.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate|scan|finalize|assign|bpr" -c 20 --csv python bench.py --workload C3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c3.csv 2>/dev/null; echo ncu rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate|scan|finalize|assign" -c 12 --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_tgt.csv 2>/dev/null; echo ncu rc=$?
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/tgt$i.json 2>/dev/null
python -c "import json;d=json.loads(open('$O/tgt$i.json').read().strip().splitlines()[-1]);r=d['roofline'];print('tgt', d['value'], d['ms_per_step'], d['phases_ms']['gate'], d['phases_ms']['assign'], r['achieved'], r.get('gemm_effective_sm_mhz'), d['clocks']['sm_mhz'])"; done
