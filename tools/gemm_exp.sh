# GEMM epilogue experiments: build variants of libmoe_b200.so with experiment defines and run the
# TGT bench phase breakdown with each (MOE_LIB_PATH). Timing only: NO_MASK / NO_CERT variants
# compute wrong gradients. Build here (CPU): bash tools/gemm_exp.sh build; on the box: ... run
cd ${GRAFT_REPO_ROOT:-/root/repo}
VARS=${GEXP_VARS:-"base: nomask:-DMOE_EXP_NO_MASK"}
if [ "$1" = build ]; then
  for v in $VARS; do
    tag=${v%%:*}; flags=$(echo ${v#*:} | tr '+' ' ')
    MOE_BUILD_DIR=/tmp/moe_var_$tag MOE_LIB_OUT=paper_2206_03382_b200/var_$tag.so MOE_NVCC_EXTRA="$flags" \
      python -m paper_2206_03382_b200.build > /dev/null || echo "build $tag failed"
    echo "built $tag ($flags)"
  done
elif [ "$1" = ncu ]; then
  # per-cycle view, each variant's GEMM launches of one step replayed alone
  mkdir -p gpurun_out/gexp
  for v in $VARS; do
    tag=${v%%:*}
    MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_$tag.so timeout 600 ncu --clock-control none -k regex:gemm_bf16 -s 60 -c 6 \
      --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,smsp__issue_active.avg.pct_of_peak_sustained_active \
      --csv python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/gexp/ncu_$tag.csv 2>/dev/null
    echo "ncu $tag rc=$?"
    python tools/ncu_gemm_table.py gpurun_out/gexp/ncu_$tag.csv $tag
  done
else
  mkdir -p gpurun_out/gexp
  for rep in 1 2; do
    for v in $VARS; do
      tag=${v%%:*}
      MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_$tag.so timeout 300 python bench.py ${GEXP_ARGS} --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/gexp/$tag.$rep.json 2>/dev/null
      python -c "import json;d=json.loads(open('gpurun_out/gexp/$tag.$rep.json').read().strip().splitlines()[-1]);p=d['phases_ms'];print('$tag', round(d['ms_per_step'],4), {k:p[k] for k in ('gate','assign','gemm_up','gemm_down','gemm_dgrad_mask','gemm_dgrad','gemm_wgrad1','gemm_wgrad2','relu_fixup')}, d['clocks']['sm_mhz'])"
    done
  done
fi
