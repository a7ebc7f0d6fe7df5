# A/B of library variants at TGV 256^3 and the 256x256x32 slab: bash tools/gpu_ab_sizes.sh v1 v2 ...
mkdir -p gpurun_out
for v in "$@"; do
  L=$PWD/paper_2207_01173_b200/libhgks_$v.so
  for args in "" "--weak"; do
    HGKS_LIB=$L timeout 300 python bench.py $args --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/abs_$v.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/abs_$v.json').read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']
print('$v', d['config']['grid'], 'fp64 %.1fM fp32 %.1fM' % (d['value']/1e6, d['fp32']['value']/1e6), 'flux %.2f/%.2f/%.2f recon %.2f' % (k['flux_x'], k['flux_y'], k['flux_z'], k['recon']))"
  done
done
