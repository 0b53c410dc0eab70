cd $GRAFT_REPO_ROOT
N=2
O=gpurun_out/vw2
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_ops.py tests/test_gpu_gate_tc.py -m gpu -x -q > $O/pytest1.log 2>&1; echo "single rc=$?"; tail -1 $O/pytest1.log
timeout 900 $TR --master-port 29611 tools/mp_parity.py > $O/mp.log 2>&1; echo "mp rc=$?"; grep -c PASS $O/mp.log; grep FAIL $O/mp.log | head -3
timeout 900 $TR --master-port 29612 tools/mp_parity_c4.py > $O/c4.log 2>&1; echo "c4 rc=$?"; grep -E "FAIL|ALL PASS" $O/c4.log
for a in peer nccl; do
  timeout 600 $TR --master-port 29613 bench.py --gpus $N --a2a $a --no-cpu-baseline > $O/b_$a.json 2> $O/b_$a.err
  python -c "import json;d=json.loads(open('$O/b_$a.json').read().strip().splitlines()[-1]);p=d['phases_ms'];print('$a', d['value'], d['ms_per_step'], p['decode'], p['encode_bwd'], p['gate'], d['clocks']['sm_mhz'], d['e2e']['value'])"
done
MOE_DISPATCH=fused timeout 600 $TR --master-port 29614 bench.py --gpus $N --no-cpu-baseline --no-e2e > $O/b_fd.json 2> $O/b_fd.err
python -c "import json;d=json.loads(open('$O/b_fd.json').read().strip().splitlines()[-1]);p=d['phases_ms'];print('fused', d['value'], d['ms_per_step'], p['encode'], p['decode_bwd'])"
