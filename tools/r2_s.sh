cd $GRAFT_REPO_ROOT
O=gpurun_out/r2s
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_layer.py tests/test_gpu_guard.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 300 python bench.py > $O/tgt.json 2> $O/tgt.err; echo "tgt rc=$?"
python -c "import json;d=json.loads(open('$O/tgt.json').read().strip().splitlines()[-1]);print('tgt', d['value'], d['ms_per_step'], d['phases_ms'], d['roofline'], d['clocks'], d['e2e']['value'])"
bash tools/ncu_wl.sh TGT 14 300
