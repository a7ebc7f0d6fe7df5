bash tools/gpu_ab2.sh "tests/test_gpu_parity.py tests/test_gpu_channel.py" pf1 default pf1 default
