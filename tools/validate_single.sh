# Single-GPU round-end evidence: every workload's bench line (device-clock GEMM spans), the
# reference arm, the in-place weight update line, and (with FULL=1) the whole single-GPU suite.
cd $GRAFT_REPO_ROOT
O=gpurun_out/vsingle
mkdir -p $O
if [ "$FULL" = 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
fi
for w in TGT C1 C2 C3; do
  timeout 400 python bench.py --workload $w > $O/$w.json 2> $O/$w.err; echo "$w rc=$?"
  python -c "import json;d=json.loads(open('$O/$w.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$w', d['value'], d['ms_per_step'], r['frac'], r.get('achieved_event_timed'), r['achieved'], d['clocks']['sm_mhz'], d['e2e']['value'], d['cpu_baseline'] and d['cpu_baseline'].get('value'))"
done
timeout 600 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"; tail -c 600 $O/ref.json
timeout 300 python bench.py --update-weights --no-cpu-baseline --no-e2e > $O/tgt_uw.json 2> $O/tgt_uw.err; echo "uw rc=$?"
python -c "import json;d=json.loads(open('$O/tgt_uw.json').read().strip().splitlines()[-1]);print('uw', d['value'], d['ms_per_step'], d['phases_ms']['weight_stats'])"
