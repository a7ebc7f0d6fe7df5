#!/bin/bash
# A/B of library variants (TGV 256^3 and the 256x256x32 slab), plus parity tests of the default build.
# usage: bash tools/gpu_ab2.sh "<pytest args or empty>" v1 v2 ...   (libhgks_<v>.so; "default" = libhgks.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T="$1"; shift
if [ -n "$T" ]; then eval timeout 1200 python -m pytest $T -x -q --timeout 300 > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log; tail -3 gpurun_out/ab_pytest.log; fi
for v in "$@"; do
  if [ "$v" = default ]; then L=$PWD/paper_2207_01173_b200/libhgks.so; else L=$PWD/paper_2207_01173_b200/libhgks_$v.so; fi
  for args in "" "--weak"; do
    HGKS_LIB=$L timeout 300 python bench.py $args --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/abs_$v$args.json 2>gpurun_out/abs_$v$args.err
    python -c "
import json; d=json.loads(open('gpurun_out/abs_$v$args.json').read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']; k2=d['fp32']['kernel_ms_per_step']
print('$v', d['config']['grid'], 'fp64 %.1fM fp32 %.1fM' % (d['value']/1e6, d['fp32']['value']/1e6), 'flux64 %.2f/%.2f/%.2f recon %.2f upd %.2f' % (k['flux_x'], k['flux_y'], k['flux_z'], k['recon'], k['update']), 'flux32 %.2f/%.2f/%.2f' % (k2['flux_x'], k2['flux_y'], k2['flux_z']), 'frac64 %.3f frac32 %.3f' % (d['roofline'].get('frac',0), d['fp32']['roofline'].get('frac',0)))" || tail -3 gpurun_out/abs_$v$args.err
  done
done
