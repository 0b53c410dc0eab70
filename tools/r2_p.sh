cd $GRAFT_REPO_ROOT
O=gpurun_out/r2q
mkdir -p $O
timeout 120 python tools/t5smoke.py > $O/smoke.log 2>&1; echo "smoke rc=$?"; cat $O/smoke.log | tail -5
timeout 600 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_layer.py -m gpu -x -q -s > $O/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "gate_fixups|passed|failed|Error" $O/pytest.log | tail -4
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/tgt.json 2> $O/tgt.err; echo "tgt rc=$?"
python -c "import json;d=json.loads(open('$O/tgt.json').read().strip().splitlines()[-1]);print('tgt', d['value'], d['ms_per_step'], d['phases_ms']['gate'], d['clocks']['sm_mhz'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate|scan|finalize|assign" -c 12 --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.csv 2>/dev/null; echo "ncu rc=$?"
