# ncu evidence for the fp32 layer (configs[0], C1): launch list of a short bench run and one
# --set full capture of the DMMA fp32 GEMM. Outputs under gpurun_out/c1/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c1
timeout 300 python bench.py --workload C1 --steps 3 --warmup 3 > gpurun_out/c1/bench.json 2> gpurun_out/c1/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/c1/launches.csv python bench.py --workload C1 --steps 2 --warmup 3 \
  > gpurun_out/c1/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_f32 -s 10 -c 5 \
  -o gpurun_out/c1/prof python bench.py --workload C1 --steps 2 --warmup 3 \
  > gpurun_out/c1/ncu_full.log 2>&1; echo "ncu full rc=$?"
