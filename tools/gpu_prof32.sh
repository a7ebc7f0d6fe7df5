mkdir -p gpurun_out
TAG=${1:-f32}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flux_kernel -s 0 -c 3 -o gpurun_out/prof_$TAG python bench.py --n 128 --steps 1 --warmup 1 --only-fp32 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
cp paper_2207_01173_b200/libhgks.so gpurun_out/libhgks_$TAG.so
