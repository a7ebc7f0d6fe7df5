# quick GPU iteration: parity tests, bench at 256^3, ncu full of the flux kernels at 128^3
mkdir -p gpurun_out
TAG=${1:-iter}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1]);print('fp64', d['value'], d['ms_per_step'], 'fp32', d['fp32']['value'], d['kernel_ms_per_step'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flux_kernel -s 3 -c 4 -o gpurun_out/prof_$TAG python bench.py --n 128 --steps 1 --warmup 1 --no-fp32 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
