# compute-sanitizer over the hot path (VERDICT r1 "sanitize the hot path"). Logs in
# gpurun_out/san/. Usage: bash tools/sanitize.sh [single|multi]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
MODE=${1:-single}
if [ "$MODE" = single ]; then
  for tool in memcheck synccheck racecheck; do
    for shape in small tgt; do
      [ $tool = racecheck ] && [ $shape = tgt ] && continue   # racecheck: small shape only (cost)
      timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 \
        python tools/sanitize_step.py --shape $shape > gpurun_out/san/${tool}_${shape}.log 2>&1
      echo "$tool $shape rc=$?"; tail -2 gpurun_out/san/${tool}_${shape}.log
    done
  done
  timeout 900 $CS --tool initcheck --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_step.py --shape small > gpurun_out/san/initcheck_small.log 2>&1
  echo "initcheck small rc=$?"; tail -2 gpurun_out/san/initcheck_small.log
else
  for tool in memcheck synccheck; do
    timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 --target-processes all \
      python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29561 tools/sanitize_step.py --shape c4s > gpurun_out/san/${tool}_c4s_w2.log 2>&1
    echo "$tool c4s W=2 rc=$?"; tail -3 gpurun_out/san/${tool}_c4s_w2.log
  done
fi
