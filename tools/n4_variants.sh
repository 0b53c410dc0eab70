# N = 4 bench variants (C4 per GPU): adaptive degree, fixed degrees, fused dispatch.
cd $GRAFT_REPO_ROOT
O=gpurun_out/n4var
mkdir -p $O
N=${N:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
i=0
run() {  # tag, env, args
  i=$((i+1))
  env $2 timeout 600 $TR --master-port $((29600+i)) bench.py --gpus $N --no-cpu-baseline --no-e2e $3 > $O/$1.json 2> $O/$1.err
  python -c "import json;d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]);p=d['phases_ms'];print('$1', round(d['value']/1e6,2), round(d['ms_per_step'],3), d['config'].get('degree'), p['gemm_up'], p['gemm_dgrad_mask'], p['encode'], p['decode_bwd'], (d.get('a2a') or {}).get('dispatch_gbs'), d['clocks']['reasons'])"
}
if [ "$SET" = final ]; then
  run copy "X=1" ""
  run fused "MOE_DISPATCH=fused" ""
  run nccl "X=1" "--a2a nccl"
  run copy_b "X=1" ""
  run fused_b "MOE_DISPATCH=fused" ""
  exit 0
fi
if [ "$SET" = parts ]; then
  run p332 "X=1" "--degree 1"
  run p224 "MOE_PARTS=2,2,4" "--degree 1"
  run p2222 "MOE_PARTS=2,2,2,2" "--degree 1"
  run p1x8 "MOE_PARTS=1,1,1,1,1,1,1,1" "--degree 1"
  run p332b "X=1" "--degree 1"
  run p224b "MOE_PARTS=2,2,4" "--degree 1"
  exit 0
fi
if [ "$SET" = adaptive ]; then
  run adaptive_a "X=1" ""
  run d1 "X=1" "--degree 1"
  run adaptive_b "X=1" ""
  run adaptive_c "X=1" ""
  exit 0
fi
run adaptive "X=1" ""
run d1 "X=1" "--degree 1"
run d2 "X=1" "--degree 2"
run d4 "X=1" "--degree 4"
run fused "MOE_DISPATCH=fused" ""
run fused_d2 "MOE_DISPATCH=fused" "--degree 2"
run adaptive2 "X=1" ""
