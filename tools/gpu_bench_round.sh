# Bench pass of a measurement round (after tools/gpu_counters_round.sh has refreshed profiles/flux_flops.json):
# the default bench line, the reference arm, config 2 (TGV 128^3), config 4 (channel H2), the P = 8 slab and the
# config-5 weak unit, and a 2-rank loopback + nccl-self dry run.
set -x
mkdir -p gpurun_out
TAG=${1:-r2b}
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; echo ref rc=$?
timeout 900 python bench.py --n 128 --no-cpu > gpurun_out/bench_tgv128_$TAG.json 2> gpurun_out/bench_tgv128_$TAG.err; echo tgv128 rc=$?
timeout 900 python bench.py --workload channel --no-cpu > gpurun_out/bench_channel_$TAG.json 2> gpurun_out/bench_channel_$TAG.err; echo channel rc=$?
timeout 900 python bench.py --weak --n 256 --no-cpu --no-e2e > gpurun_out/bench_slab_$TAG.json 2> gpurun_out/bench_slab_$TAG.err; echo slab rc=$?
timeout 900 python bench.py --weak --n 512 --no-cpu --no-e2e --steps 4 > gpurun_out/bench_weak512_$TAG.json 2> gpurun_out/bench_weak512_$TAG.err; echo weak512 rc=$?
timeout 900 python bench.py --gpus 2 --transport loopback --weak --n 512 --no-cpu --no-e2e --steps 4 > gpurun_out/bench_loop2_$TAG.json 2> gpurun_out/bench_loop2_$TAG.err; echo loop2 rc=$?
timeout 900 python bench.py --transport nccl-self --no-cpu --no-e2e --steps 4 > gpurun_out/bench_ncclself_$TAG.json 2> gpurun_out/bench_ncclself_$TAG.err; echo ncclself rc=$?
