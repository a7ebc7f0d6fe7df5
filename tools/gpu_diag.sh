bash tools/gpu_variants.sh libhgks_tpb1.so libhgks.so libhgks_tpb4.so
for t in 1 2 4; do HGKS_LIB=$PWD/paper_2207_01173_b200/libhgks_timing$t.so python tools/phase_timing.py 256; done
