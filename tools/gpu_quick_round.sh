# Quick measurement round of the current build: counters (for flux_flops.json), pytest -m gpu, smoke,
# default bench line.  usage: bash tools/gpu_quick_round.sh TAG
TAG=${1:-r2g}
bash tools/gpu_counters_round.sh $TAG
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.json | cut -c1-400
