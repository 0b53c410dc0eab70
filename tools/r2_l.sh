cd $GRAFT_REPO_ROOT
O=gpurun_out/r2l
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest.log
timeout 300 python bench.py --no-cpu-baseline > $O/tgt.json 2> $O/tgt.err; echo "tgt rc=$?"
timeout 300 python bench.py --workload C3 --no-cpu-baseline > $O/c3.json 2> $O/c3.err; echo "c3 rc=$?"
for f in tgt c3; do python -c "import json;d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]);print('$f', d['value'], d['ms_per_step'], d['phases_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gate_tc|gate_fixup" -s 6 -c 2 -o $O/gate python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate|scan|finalize|assign|bpr|decode|encode" -c 40 --csv python bench.py --workload C3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c3.csv 2> $O/ncu_c3.err; echo "ncu c3 rc=$?"
