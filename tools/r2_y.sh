cd $GRAFT_REPO_ROOT
O=gpurun_out/r2y
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_layer.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 300 python bench.py --no-cpu-baseline > $O/tgt.json 2> $O/tgt.err
python -c "import json;d=json.loads(open('$O/tgt.json').read().strip().splitlines()[-1]);r=d['roofline'];print('tgt', d['value'], d['ms_per_step'], d['phases_ms']['gate'], r['achieved'], r.get('gemm_effective_sm_mhz'), d['clocks'])"
bash tools/ncu_wl.sh C3 17 300
