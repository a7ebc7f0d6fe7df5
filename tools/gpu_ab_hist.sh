#!/bin/bash
# A/B of library variants on the per-step diagnostic history cost (bench aux history_ms_per_step) plus the
# GPU diagnostics tests of the default build.  usage: bash tools/gpu_ab_hist.sh v1 v2 ...  ("default" = libhgks.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_diagnostics.py -q -x > gpurun_out/diag_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/diag_pytest.log
for v in "$@"; do
  if [ "$v" = default ]; then L=$PWD/paper_2207_01173_b200/libhgks.so; else L=$PWD/paper_2207_01173_b200/libhgks_$v.so; fi
  HGKS_LIB=$L timeout 300 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/abh_$v.json 2>gpurun_out/abh_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/abh_$v.json').read().strip().splitlines()[-1])
print('$v', 'fp64 %.1fM fp32 %.1fM' % (d['value']/1e6, d['fp32']['value']/1e6), 'aux', d['aux_ms'], 'upd', d['kernel_ms_per_step']['update'])"
done
