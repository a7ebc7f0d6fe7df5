#!/bin/bash
# ncu --set full (with source) of the flux kernels at 128^3 fp64 (stage 1, x and y) for the current build
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${1:-ring}; K=${2:-flux}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 0 -c 2 -o gpurun_out/prof_$TAG python bench.py --n 128 --steps 1 --warmup 1 --no-fp32 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
cp paper_2207_01173_b200/libhgks.so gpurun_out/libhgks_$TAG.so
