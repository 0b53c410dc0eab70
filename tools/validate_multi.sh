# Round-2 multi-GPU validation at N = 4: every multi-GPU test (full-shape C4 parity +
# invariance on both transports and the fused dispatch, the bounds-checked C4 run at W = 2,
# small-shape mp_parity, scenarios), bench lines (copy engines, NCCL), the capacity x degree sweep.
cd $GRAFT_REPO_ROOT
N=4
O=gpurun_out/vmulti
mkdir -p $O
./tools/probe/gtimer > $O/gtimer.txt 2>&1; cat $O/gtimer.txt
timeout 2400 python -m pytest tests/test_gpu_multi.py -x -q -s > $O/pytest_multi.log 2>&1; echo "multi rc=$?"
grep -E "PASS|FAIL|passed|failed" $O/pytest_multi.log | tail -60 | cut -c1-220
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29581 bench.py --gpus $N > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 $TR --master-port 29582 bench.py --gpus $N --a2a nccl --no-cpu-baseline > $O/bench_nccl.json 2> $O/bench_nccl.err; echo "bench nccl rc=$?"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TR2 --master-port 29584 bench.py --gpus 2 --no-cpu-baseline > $O/bench_n2.json 2> $O/bench_n2.err; echo "bench n2 rc=$?"
timeout 600 $TR --master-port 29585 bench.py --gpus $N --impl reference > $O/ref_n4.json 2> $O/ref_n4.err; echo "ref n4 rc=$?"
for f in bench bench_nccl bench_n2; do python -c "import json;d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]);print('$f', d['value'], d['ms_per_step'], d['clocks'], d.get('a2a',{}).get('dispatch_gbs'), d['e2e']['value'])"; done
if [ "$SWEEP" != 0 ]; then
  timeout 1500 $TR --master-port 29583 tools/sweep.py --out $O/sweep_n4.json > $O/sweep.log 2>&1; echo "sweep rc=$?"; tail -5 $O/sweep.log
fi
