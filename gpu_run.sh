cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench2.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
