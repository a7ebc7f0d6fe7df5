mkdir -p gpurun_out
for v in "$@"; do
  HGKS_LIB=$PWD/paper_2207_01173_b200/$v timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_var_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_var_$v.log').read().strip().splitlines()[-1]);print('$v', 'fp64 %.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], 'fp32 %.4g'%d['fp32']['value'], {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
done
