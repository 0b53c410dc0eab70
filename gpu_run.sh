cd $GRAFT_REPO_ROOT
echo "== 3 stages, 2 epi bufs"; timeout 300 python tools/gemm_bench.py 2>&1 | tail -3
echo "== 4 stages, 1 epi buf"; MOE_LIB_PATH=gpurun_out/libmoe_v41.so timeout 300 python tools/gemm_bench.py 2>&1 | tail -3
echo "== 2 stages, 2 epi bufs"; MOE_LIB_PATH=gpurun_out/libmoe_v42.so timeout 300 python tools/gemm_bench.py 2>&1 | tail -3
