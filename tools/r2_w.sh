cd $GRAFT_REPO_ROOT
N=4
O=gpurun_out/r2w
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for sp in 1 2 4 1 2 4; do
  MOE_CE_SPLIT=$sp timeout 600 $TR --master-port 2959$sp bench.py --gpus $N --no-cpu-baseline --no-e2e > $O/b_$sp.json 2> $O/b_$sp.err
  python -c "import json;d=json.loads(open('$O/b_$sp.json').read().strip().splitlines()[-1]);a=d['a2a'];print('split=$sp', d['value'], d['ms_per_step'], a.get('dispatch_gbs'), a.get('dispatch_xfer_ms_per_step'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
MOE_CE_SPLIT=4 timeout 900 $TR --master-port 29599 tools/mp_parity_c4.py --degrees 1,2 > $O/c4_split4.log 2>&1; echo "c4 split4 rc=$?"; grep -E "PASS|FAIL" $O/c4_split4.log | cut -c1-150
