# ncu evidence for one bench workload: launch list of a short bench run and one --set full
# capture of one step's launches. Usage: bash tools/ncu_wl.sh WORKLOAD NLAUNCH [SKIP]
# Outputs under gpurun_out/ncu_<workload>/.
cd $GRAFT_REPO_ROOT
WL=${1:-TGT}; N=${2:-17}; S=${3:-300}
O=gpurun_out/ncu_$WL
mkdir -p $O
B="bench.py --workload $WL --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 python $B > $O/bench.json 2> $O/bench.err; echo "bench $WL rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches.csv python $B > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -s $S -c $N \
  -o $O/prof python $B > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
