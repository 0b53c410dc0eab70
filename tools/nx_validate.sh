# Multi-GPU check (NGPU, default 2) of the driver's scaling launch: both bench arms under torchrun at N=NGPU.
# Outputs under gpurun_out/n${NGPU:-2}/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/n${NGPU:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NGPU:-2} --master-addr 127.0.0.1"
timeout 400 $R --master-port 29511 bench.py --gpus ${NGPU:-2} --impl reference --steps 3 --warmup 3 \
  > gpurun_out/n${NGPU:-2}/ref.json 2> gpurun_out/n${NGPU:-2}/ref.err; echo "ref rc=$?"
timeout 600 $R --master-port 29512 bench.py --gpus ${NGPU:-2} > gpurun_out/n${NGPU:-2}/bench.json 2> gpurun_out/n${NGPU:-2}/bench.err; echo "bench rc=$?"
