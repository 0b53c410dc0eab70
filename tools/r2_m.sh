cd $GRAFT_REPO_ROOT
export GEXP_VARS="base: actmask:-DMOE_EXP_NO_MASK+-DMOE_EXP_ACT_MASK fix1:-DMOE_FIX_TOK=1 splitacc:-DMOE_GATE_SPLIT_ACC"
bash tools/gemm_exp.sh run
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_layer.py -m gpu -x -q -k "bpr or BPR or gating or C3 or full_size or weight_stats" > gpurun_out/gexp/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gexp/pytest.log
MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_base.so timeout 300 python bench.py --workload C3 --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/gexp/c3.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/gexp/c3.json').read().strip().splitlines()[-1]);print('c3', d['value'], d['ms_per_step'], d['phases_ms'])"
