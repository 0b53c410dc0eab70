# relu_fixup variants: ncu per launch (isolated) + the layer tests on the default build.
cd $GRAFT_REPO_ROOT
O=gpurun_out/fixup_ab
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layer.py -q -x 2>&1 | tail -1
for v in ${VARS:-f32p f64p cta4}; do
  MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_$v.so timeout 300 ncu --clock-control none -k regex:"relu_fixup" -s 5 -c 5 \
    --metrics gpu__time_duration.sum --csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$v.csv 2>/dev/null
  echo "$v $(grep relu_fixup $O/ncu_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
