mkdir -p gpurun_out
bash tools/gpu_ab.sh head hf
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_b1.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_b1.log
timeout 900 python tools/precision_twin.py --n 128 --t-end 20 --every 0.25 --out gpurun_out/twin128.json > gpurun_out/twin128.log 2>&1; echo twin rc=$?; tail -2 gpurun_out/twin128.log
timeout 900 python tools/tgv_budget.py --n 128 --t-end 10 --every 0.1 --out gpurun_out/budget128.json > gpurun_out/budget128.log 2>&1; echo budget rc=$?; tail -5 gpurun_out/budget128.log
