# A/B of the certified gate kernel: var_old.so (parent commit) vs var_new.so, ncu per launch, plus
# the gate tests on the current build.
cd $GRAFT_REPO_ROOT
O=gpurun_out/gate_ab
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_layer.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for v in old new; do
  MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_$v.so timeout 300 ncu --clock-control none -k regex:"gate_tc5|gate_fixup" -s 10 -c 6 \
    --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv \
    python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$v.csv 2>/dev/null
  echo "ncu $v rc=$?"
  grep -E "gate_tc5|gate_fixup" $O/ncu_$v.csv | awk -F'","' '{print "'$v'", $5, $(NF-2), $NF}' | cut -c1-150
done
