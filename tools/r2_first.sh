cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2a
nvidia-smi -L > gpurun_out/r2a/gpus.txt; nproc >> gpurun_out/r2a/gpus.txt; free -g >> gpurun_out/r2a/gpus.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/r2a/pytest_multi.log 2>&1; echo "multi rc=$?"
timeout 300 python bench.py > gpurun_out/r2a/bench1.json 2> gpurun_out/r2a/bench1.err; echo "bench1 rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/r2a/bench2.json 2> gpurun_out/r2a/bench2.err; echo "bench2 rc=$?"
