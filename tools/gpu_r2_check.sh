#!/bin/bash
# One GPU call: ALU peaks microbench, GPU tests, default bench line, loopback 2-rank bench line.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/alu_peaks tools/microbench/alu_peaks.cu && /tmp/alu_peaks > gpurun_out/alu_peaks.json
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --gpus 2 --transport loopback --no-cpu > gpurun_out/bench_lb2.json 2> gpurun_out/bench_lb2.err
tail -3 gpurun_out/pytest_gpu.log
