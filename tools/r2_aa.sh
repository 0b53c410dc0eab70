cd $GRAFT_REPO_ROOT
O=gpurun_out/r2aa
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_guard.py tests/test_gpu_gate_tc.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for d in 1 0 1 0; do
  MOE_DEFER_FIXUP=$d timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/b$d.json 2>/dev/null
  python -c "import json;d=json.loads(open('$O/b$d.json').read().strip().splitlines()[-1]);p=d['phases_ms'];print('defer=$d', d['value'], d['ms_per_step'], p['gemm_down'], p['relu_fixup'], d['roofline'].get('gemm_effective_sm_mhz'), d['clocks']['sm_mhz'])"
done
MOE_DEFER_FIXUP=1 timeout 300 python bench.py --workload C3 --no-cpu-baseline --no-e2e > $O/c3.json 2>/dev/null
python -c "import json;d=json.loads(open('$O/c3.json').read().strip().splitlines()[-1]);p=d['phases_ms'];print('c3', d['value'], d['ms_per_step'], p['relu_fixup'], d['clocks']['sm_mhz'])"
