bash tools/gpu_ab2.sh "tests/test_gpu_parity.py tests/test_gpu_forcing.py tests/test_gpu_channel_physics.py" cf default u1
