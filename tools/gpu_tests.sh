mkdir -p gpurun_out
TAG=${1:-t}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1]);print('fp64', d['value'], d['ms_per_step'], 'fp32', d['fp32']['value'], d['roofline'].get('frac'))"
