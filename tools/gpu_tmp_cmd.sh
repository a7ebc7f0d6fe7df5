bash tools/gpu_ab2.sh "" default rm8 rm10 default rm8
