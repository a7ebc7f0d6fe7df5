# Whole measurement round on one box: counters (refreshes nothing here: run tools/counters_to_profile.py
# locally after), full GPU test suite, smoke.  usage: bash tools/gpu_round_all.sh TAG
TAG=${1:-r2c}
bash tools/gpu_counters_round.sh $TAG
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
# compute-sanitizer: closed on the GPU pool since the end of round 2 (tools/gpu_sanitize.sh for pools that allow it)
