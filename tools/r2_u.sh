cd $GRAFT_REPO_ROOT
O=gpurun_out/r2u
mkdir -p $O
for pdl in 1 0 1 0; do
  MOE_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/pdl$pdl.json 2>/dev/null
  python -c "import json;d=json.loads(open('$O/pdl$pdl.json').read().strip().splitlines()[-1]);r=d['roofline'];print('pdl=$pdl', d['value'], d['ms_per_step'], r['achieved'], r.get('gemm_span_ms_per_step'), d['clocks']['sm_mhz'])"
done
