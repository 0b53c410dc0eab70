# Single-GPU round check: gate / layer tests, TGT bench (+ --update-weights variant), C3 bench,
# C3 ncu launch list + one-step --set full capture.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2j
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_layer.py -m gpu -x -q -s > $O/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "gate_fixups|passed|failed|Error" $O/pytest.log | tail -4
timeout 300 python bench.py > $O/tgt.json 2> $O/tgt.err; echo "tgt rc=$?"
timeout 300 python bench.py --update-weights --no-cpu-baseline > $O/tgt_uw.json 2> $O/tgt_uw.err; echo "tgt uw rc=$?"
timeout 300 python bench.py --workload C3 --no-cpu-baseline > $O/c3.json 2> $O/c3.err; echo "c3 rc=$?"
for f in tgt tgt_uw c3; do python -c "import json;d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]);print('$f', d['value'], d['ms_per_step'], d['phases_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
bash tools/ncu_wl.sh C3 19 300
