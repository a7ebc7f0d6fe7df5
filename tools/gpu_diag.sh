./tools/microbench/fp64_pipes; nvidia-smi --query-gpu=clocks.sm --format=csv
