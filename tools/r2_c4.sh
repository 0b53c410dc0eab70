# C4 full-shape parity + strategy invariance at W = $1, and the weight-update tests on GPU 0.
cd $GRAFT_REPO_ROOT
W=${1:-2}
mkdir -p gpurun_out/r2c4
timeout 600 python -m pytest tests/test_gpu_layer.py -q -k "in_place or expert_grads or set_weights" > gpurun_out/r2c4/pytest_weights.log 2>&1; echo "weights rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29533 tools/mp_parity_c4.py > gpurun_out/r2c4/c4_w$W.log 2>&1; echo "c4 rc=$?"
tail -20 gpurun_out/r2c4/c4_w$W.log
