cd $GRAFT_REPO_ROOT
O=gpurun_out/r2gate3
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_layer.py -m gpu -x -q -s > $O/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "gate_fixups|passed|failed|Error" $O/pytest.log | tail -8
timeout 300 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gate_tc|gate_fixup" -s 6 -c 2 -o $O/gate python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1; echo "ncu rc=$?"
