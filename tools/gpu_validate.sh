# Round-end validation on one B200: GPU tests, smoke, the default bench line, every single-GPU
# BASELINE config, and the reference arm. Outputs under gpurun_out/val/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/val
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/val/pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/val/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/val/bench.json 2> gpurun_out/val/bench.err; echo "bench rc=$?"
for w in C1 C2 C3; do
  timeout 400 python bench.py --workload $w --steps 30 > gpurun_out/val/$w.json 2> gpurun_out/val/$w.err; echo "$w rc=$?"
done
timeout 600 python bench.py --impl reference > gpurun_out/val/ref.json 2> gpurun_out/val/ref.err; echo "ref rc=$?"
