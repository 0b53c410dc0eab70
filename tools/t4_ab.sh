cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_ops.py -q -x 2>&1 | tail -2
export GEXP_VARS="t3: t4:"
bash tools/gemm_exp.sh ncu
bash tools/gemm_exp.sh run
