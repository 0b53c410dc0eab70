# Multi-GPU validation at N = $1 GPUs: every multi-GPU test (incl. full-shape C4 parity and
# strategy invariance) and the N-GPU bench line.
cd $GRAFT_REPO_ROOT
N=${1:-4}
mkdir -p gpurun_out/r2m$N
timeout 2400 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/r2m$N/pytest_multi.log 2>&1; echo "multi rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N > gpurun_out/r2m$N/bench.json 2> gpurun_out/r2m$N/bench.err; echo "bench rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r2m$N/pytest_multi.log | tail -40
