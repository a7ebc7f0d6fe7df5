mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu2.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu2.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench256.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/bench256.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-fp32 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flux_kernel -s 3 -c 2 -o gpurun_out/prof_flux_r1 python bench.py --n 128 --steps 1 --warmup 1 --no-fp32 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu_full.log
