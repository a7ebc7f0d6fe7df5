bash tools/gpu_ab2.sh "" default f4 default f4
