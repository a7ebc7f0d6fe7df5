# Re-entry verification: GPU parity suite, smoke(), default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_verify.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_verify.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu_verify.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_verify.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/smoke_verify.log
timeout 900 python bench.py > gpurun_out/bench_verify.json 2> gpurun_out/bench_verify.err; echo bench rc=$?
tail -1 gpurun_out/bench_verify.json
