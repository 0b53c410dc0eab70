# Single-GPU check: the named test files (or all -m gpu tests), then the default bench line.
cd $GRAFT_REPO_ROOT
TAG=${1:-r2s}
shift
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest ${@:-tests} -m gpu -x -q > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/$TAG/pytest.log
timeout 300 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/$TAG/bench.err
