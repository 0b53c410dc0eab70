cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_tgt.json 2> gpurun_out/bench_tgt.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16|encode_kernel|decode_kernel|gate_dmma|encode_bwd|decode_bwd|relu_fixup|scan_kernel|assign_kernel" -s 17 -c 17 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -2 gpurun_out/ncu_full.log
