cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tools/mp_parity.py > gpurun_out/mp$N.log 2>&1; echo "mp rc=$?"
grep -cE "PASS" gpurun_out/mp$N.log; grep -E "FAIL" gpurun_out/mp$N.log | head -3
for n in 2 $N; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo "bench n=$n rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_n$n.json')); print(d['value'], d['ms_per_step'], d['config']['degree'], d['roofline']['frac'], d['e2e']['value'], {k:v for k,v in d['phases_ms'].items() if v})"
done
