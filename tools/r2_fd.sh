# Fused-dispatch A/B at N GPUs: parity (mp_parity incl. peer-fd cases, full-shape C4 incl. peer-fd
# invariance), then the C4 bench line with copy-engine dispatch and with MOE_DISPATCH=fused.
cd $GRAFT_REPO_ROOT
N=${1:-2}
O=gpurun_out/r2fd$N
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29571 tools/mp_parity.py > $O/mp_parity.log 2>&1; echo "mp_parity rc=$?"
grep -E "FAIL|peer-fd" $O/mp_parity.log | head
timeout 900 $TR --master-port 29572 tools/mp_parity_c4.py > $O/c4.log 2>&1; echo "c4 rc=$?"
grep -E "PASS|FAIL" $O/c4.log | cut -c1-200
for mode in copy fused; do
  MOE_DISPATCH=$mode timeout 600 $TR --master-port 29573 bench.py --gpus $N --no-cpu-baseline > $O/bench_$mode.json 2> $O/bench_$mode.err; echo "bench $mode rc=$?"
  python -c "import json;d=json.loads(open('$O/bench_$mode.json').read().strip().splitlines()[-1]);print('$mode', d['value'], d['ms_per_step'], d['phases_ms'].get('encode'), d['phases_ms'].get('decode_bwd'), d['a2a'].get('dispatch_gbs'))"
done
