cd $GRAFT_REPO_ROOT
O=gpurun_out/r2k
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_layer.py tests/test_gpu_ops.py -m gpu -x -q -s > $O/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "gate_fixups|passed|failed|Error" $O/pytest.log | tail -4
timeout 300 python bench.py --no-cpu-baseline > $O/tgt.json 2> $O/tgt.err; echo "tgt rc=$?"
timeout 300 python bench.py --update-weights --no-cpu-baseline > $O/tgt_uw.json 2> $O/tgt_uw.err; echo "tgt uw rc=$?"
for f in tgt tgt_uw; do python -c "import json;d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]);print('$f', d['value'], d['ms_per_step'], d['phases_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate|scan|finalize|assign|weight_stats" -c 30 --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --update-weights > $O/ncu_gate.csv 2> $O/ncu.err; echo "ncu rc=$?"
