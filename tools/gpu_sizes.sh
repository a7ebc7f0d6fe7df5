# per-GPU rates at the slab sizes of the multi-GPU configs (one GPU): 256x256x32 (config 3 at P=8),
# 512x512x64 (config 5 weak unit), and 512^3 (config 5 on one GPU)
mkdir -p gpurun_out
timeout 600 python bench.py --weak --n 256 --no-e2e --no-cpu > gpurun_out/bench_weak256.json 2>/dev/null; echo weak256 rc=$?
timeout 600 python bench.py --weak --n 512 --no-e2e --no-cpu > gpurun_out/bench_weak512.json 2>/dev/null; echo weak512 rc=$?
timeout 900 python bench.py --n 512 --steps 3 --warmup 3 --no-e2e --no-cpu --no-fp32 > gpurun_out/bench_512.json 2>/dev/null; echo n512 rc=$?
for f in bench_weak256 bench_weak512 bench_512; do python -c "
import json,sys; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['config']['grid'], round(d['value']/1e6,1), 'M fp64', round(d.get('fp32',{}).get('value',0)/1e6,1), 'M fp32', round(d['ms_per_step'],2), 'ms')"; done
