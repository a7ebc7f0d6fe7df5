mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_v2.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_v2.log
for v in libhgks.so libhgks_minb1.so; do
  HGKS_LIB=$PWD/paper_2207_01173_b200/$v timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_v2_$v.log 2>&1; echo bench $v rc=$?
  python -c "import json;d=json.loads(open('gpurun_out/bench_v2_$v.log').read().strip().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['fp32']['value'], d['kernel_ms_per_step'])"
  HGKS_LIB=$PWD/paper_2207_01173_b200/$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:flux_kernel -s 3 -c 1 -o gpurun_out/prof_v2_$v python bench.py --n 128 --steps 1 --warmup 1 --no-fp32 --no-e2e --no-cpu > gpurun_out/ncu_v2_$v.log 2>&1; echo ncu rc=$?
done
