#!/bin/bash
# ncu --set full (with source) of the stage-1 x/y flux kernels at 128^3 fp64 for a library variant
# usage: bash tools/gpu_ncu_var.sh <variant|default> [kernel regex] [extra bench args]
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
V=${1:-default}; K=${2:-flux_kernel}; shift 2; EXTRA="$@"
if [ "$V" = default ]; then L=$PWD/paper_2207_01173_b200/libhgks.so; else L=$PWD/paper_2207_01173_b200/libhgks_$V.so; fi
case "$EXTRA" in *--only-fp32*) PREC="";; *) PREC="--no-fp32";; esac
HGKS_LIB=$L timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 0 -c 2 -o gpurun_out/prof_$V python bench.py --n 128 --steps 1 --warmup 1 $PREC --no-e2e --no-cpu $EXTRA > gpurun_out/ncu_$V.log 2>&1; echo ncu rc=$?
cp $L gpurun_out/libhgks_$V.so
