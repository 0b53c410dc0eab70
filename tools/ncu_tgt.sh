# ncu evidence for the TGT bench step: launch list of a short bench run and one --set full capture
# of 16 consecutive steady-state launches (one step's worth). Outputs under gpurun_out/tgt/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tgt
B="bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 python $B > gpurun_out/tgt/bench.json 2> gpurun_out/tgt/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/tgt/launches.csv python $B > gpurun_out/tgt/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -s 300 -c 16 \
  -o gpurun_out/tgt/prof python $B > gpurun_out/tgt/ncu_full.log 2>&1; echo "ncu full rc=$?"
