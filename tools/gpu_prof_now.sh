# ncu --set full of the three stage-1 flux kernels (128^3 fp64) + phase timing of the current build
mkdir -p gpurun_out
TAG=${1:-cur}
python -m paper_2207_01173_b200.build -DHGKS_PHASE_TIMING -out=libhgks_timing.so > /dev/null 2>&1
timeout 300 python tools/phase_timing.py 128 > gpurun_out/phase_$TAG.log 2>&1; echo phase rc=$?; tail -2 gpurun_out/phase_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flux_kernel -s 0 -c 3 -o gpurun_out/prof_$TAG python bench.py --n 128 --steps 1 --warmup 1 --no-fp32 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
cp paper_2207_01173_b200/libhgks.so gpurun_out/libhgks_$TAG.so
