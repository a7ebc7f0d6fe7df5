# loopback-group decomposition tests + full GPU suite + NCCL same-GPU probe + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decomposition.py -q -x > gpurun_out/pytest_decomp.log 2>&1; echo decomp rc=$?
tail -15 gpurun_out/pytest_decomp.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/nccl_same_gpu.py > gpurun_out/nccl_same_gpu.log 2>&1; echo nccl rc=$?
grep -v "^\[W" gpurun_out/nccl_same_gpu.log | tail -8
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu_all.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_decomp.json 2> gpurun_out/bench_decomp.err; echo bench rc=$?
tail -1 gpurun_out/bench_decomp.json | cut -c1-400
