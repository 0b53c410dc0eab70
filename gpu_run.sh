cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/mp_parity.py > gpurun_out/mp.log 2>&1; echo "mp rc=$?"
grep -E "PASS|FAIL|Error|error|Traceback" gpurun_out/mp.log | head -20
for d in 2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$d bench.py --gpus 2 --steps 20 --warmup 5 --degree $d --no-e2e > gpurun_out/bench_n2_d$d.json 2> gpurun_out/bench_n2_d$d.err; echo "bench d=$d rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_n2_d$d.json')); print(d['value'], d['ms_per_step'], d['config']['degree'], {k:v for k,v in d['phases_ms'].items() if v})"
done
