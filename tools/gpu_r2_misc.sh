#!/bin/bash
# sanitizer runs, ncu of the reconstruction and fp32 flux kernels, config-2 (128^3) bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/gpu_sanitize.sh 2>&1 | tee gpurun_out/sanitize_summary.txt
timeout 600 ncu --set full --clock-control none -k regex:recon -s 0 -c 4 -o gpurun_out/prof_recon python bench.py --n 256 --steps 1 --warmup 1 --no-fp32 --no-e2e --no-cpu > gpurun_out/ncu_recon.log 2>&1; echo ncu recon rc=$?
bash tools/gpu_ncu_var.sh default flux_kernel --only-fp32
timeout 600 python bench.py --n 128 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_tgv128.json 2> gpurun_out/bench_tgv128.err; echo bench128 rc=$?
