cd $GRAFT_REPO_ROOT
O=gpurun_out/r2v
mkdir -p $O
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/b$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('$O/b$i.json').read().strip().splitlines()[-1]);r=d['roofline'];print('run$i', d['value'], d['ms_per_step'], r['achieved'], r.get('gemm_effective_sm_mhz'), d['clocks'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"gemm_bf16" -c 6 --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.csv 2>/dev/null; echo ncu rc=$?
