# Single-GPU round-end evidence: every workload's bench line (device-clock GEMM spans), the
# reference arm, and the gate fix-up variant A/B.
cd $GRAFT_REPO_ROOT
O=gpurun_out/vsingle
mkdir -p $O
for w in TGT C1 C2 C3; do
  timeout 400 python bench.py --workload $w > $O/$w.json 2> $O/$w.err; echo "$w rc=$?"
  python -c "import json;d=json.loads(open('$O/$w.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$w', d['value'], d['ms_per_step'], r['frac'], r.get('achieved_event_timed'), r['achieved'], d['clocks']['sm_mhz'], d['e2e']['value'], d['cpu_baseline'] and d['cpu_baseline'].get('value'))"
done
timeout 600 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"; tail -c 600 $O/ref.json
timeout 300 python bench.py --update-weights --no-cpu-baseline --no-e2e > $O/tgt_uw.json 2> $O/tgt_uw.err; echo "uw rc=$?"
python -c "import json;d=json.loads(open('$O/tgt_uw.json').read().strip().splitlines()[-1]);print('uw', d['value'], d['ms_per_step'], d['phases_ms']['weight_stats'])"
for v in base fw16; do
  MOE_LIB_PATH=$PWD/paper_2206_03382_b200/var_$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate_fixup" -c 3 --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_fix_$v.csv 2>/dev/null; echo "ncu $v rc=$?"
done
