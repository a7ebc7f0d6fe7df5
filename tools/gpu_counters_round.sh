# Counters pass of a measurement round (run BEFORE the bench lines, which read profiles/flux_flops.json):
# ncu launch list of a 2-step bench run, SASS flop / DRAM counters of the flux, reconstruction and update
# kernels (fp64 + fp32) at 256^3, and one ncu --set full capture of the stage-1 fp64 flux kernels at 128^3.
set -x
mkdir -p gpurun_out
TAG=${1:-r2b}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-fp32 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu-launch rc=$?
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none -k regex:"flux_kernel|recon_|update_kernel" -c 16 --csv --log-file gpurun_out/counters64_$TAG.csv python bench.py --steps 1 --warmup 1 --no-fp32 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu-c64 rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:"flux_kernel|recon_|update_kernel" -c 16 --csv --log-file gpurun_out/counters32_$TAG.csv python bench.py --steps 1 --warmup 1 --only-fp32 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu-c32 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flux_kernel -s 3 -c 6 -o gpurun_out/prof_full_$TAG python bench.py --n 128 --steps 1 --warmup 1 --no-fp32 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu-full rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flux_kernel -s 0 -c 3 -o gpurun_out/prof_full32_$TAG python bench.py --n 128 --steps 1 --warmup 1 --only-fp32 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu-full32 rc=$?
cp paper_2207_01173_b200/libhgks.so gpurun_out/libhgks_$TAG.so
