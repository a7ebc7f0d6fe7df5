set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "gp_flux or operator or uniform or invalid or blowup or t_end or step_parity" > gpurun_out/pytest_gpu1.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu1.log
timeout 600 python bench.py --n 128 --steps 3 --warmup 1 --no-cpu > gpurun_out/bench128.log 2>&1; echo bench rc=$?
tail -5 gpurun_out/bench128.log
