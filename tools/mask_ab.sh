# A/B of the current library against a previous build (paper_2206_03382_b200/var_old.so, built
# from the parent commit): the GEMM / gate / layer GPU tests on the current build, then the TGT
# bench alternating old / new, then the GEMM launches of one step under ncu (per-cycle view).
cd $GRAFT_REPO_ROOT
O=gpurun_out/mask
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_layer.py tests/test_gpu_ops.py tests/test_gpu_gemm.py tests/test_gpu_guard.py tests/test_gpu_gate_tc.py tests/test_gpu_checks.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for r in 1 2; do
for v in old new; do
  MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 > $O/tgt_$v$r.json 2> $O/tgt_$v$r.err
  python -c "import json;d=json.loads(open('$O/tgt_$v$r.json').read().strip().splitlines()[-1]);p=d['phases_ms'];print('$v$r', round(d['value']/1e6,2), round(d['ms_per_step'],4), p['gemm_up'], p['gemm_down'], p['gemm_dgrad_mask'], p['gemm_dgrad'], p['relu_fixup'], d['roofline']['gemm_effective_sm_mhz'])"
done; done
cp paper_2206_03382_b200/var_old.so paper_2206_03382_b200/var_o.so
GEXP_VARS="o: new:" bash tools/gemm_exp.sh ncu
