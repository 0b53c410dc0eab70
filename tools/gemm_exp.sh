# GEMM epilogue experiments: build variants of libmoe_b200.so with experiment defines and run the
# TGT bench phase breakdown with each (MOE_LIB_PATH). Timing only: NO_MASK / NO_CERT variants
# compute wrong gradients. Build here (CPU), run on the box: bash tools/gemm_exp.sh run
cd ${GRAFT_REPO_ROOT:-/root/repo}
VARS="base: nomask:-DMOE_EXP_NO_MASK nocert:-DMOE_EXP_NO_CERT nomasknocert:-DMOE_EXP_NO_MASK+-DMOE_EXP_NO_CERT up4:-DMOE_UP_EPI_WARPS=4 all8:-DMOE_EPI_WARPS=8 st5:-DMOE_GEMM_STAGES_PAIR=5"
if [ "$1" = build ]; then
  for v in $VARS; do
    tag=${v%%:*}; flags=$(echo ${v#*:} | tr '+' ' ')
    MOE_BUILD_DIR=/tmp/moe_var_$tag MOE_LIB_OUT=paper_2206_03382_b200/var_$tag.so MOE_NVCC_EXTRA="$flags" \
      python -m paper_2206_03382_b200.build > /dev/null || echo "build $tag failed"
    echo "built $tag ($flags)"
  done
else
  mkdir -p gpurun_out/gexp
  for v in $VARS; do
    tag=${v%%:*}
    for rep in 1 2; do
      MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_$tag.so timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/gexp/$tag.$rep.json 2>/dev/null
      python -c "import json;d=json.loads(open('gpurun_out/gexp/$tag.$rep.json').read().strip().splitlines()[-1]);p=d['phases_ms'];print('$tag', round(d['ms_per_step'],4), {k:p[k] for k in ('gemm_up','gemm_down','gemm_dgrad_mask','gemm_dgrad','gemm_wgrad1','gemm_wgrad2')}, d['clocks']['sm_mhz'])"
    done
  done
fi
