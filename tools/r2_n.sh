cd $GRAFT_REPO_ROOT
O=gpurun_out/r2n
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q -s > $O/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|MOE_CHECK" $O/pytest.log | tail -6
timeout 300 python bench.py > $O/tgt.json 2> $O/tgt.err; echo "tgt rc=$?"
python -c "import json;d=json.loads(open('$O/tgt.json').read().strip().splitlines()[-1]);print('tgt', d['value'], d['ms_per_step'], d['phases_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['e2e']['value'], d['cpu_baseline']['value'])"
