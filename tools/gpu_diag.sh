bash tools/gpu_variants.sh libhgks.so libhgks_t16.so
