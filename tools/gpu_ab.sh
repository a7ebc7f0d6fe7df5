# A/B timing of library variants: bash tools/gpu_ab.sh name1 name2 ...  (paper_2207_01173_b200/libhgks_<name>.so)
mkdir -p gpurun_out
for v in "$@"; do
  for rep in $(seq ${REPS:-1}); do
    HGKS_LIB=$PWD/paper_2207_01173_b200/libhgks_$v.so timeout 300 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
k = d["kernel_ms_per_step"]
k32 = d["fp32"].get("kernel_ms_per_step", {})
f = lambda k: "/".join(f"{k[x]:.2f}" for x in ("flux_x", "flux_y", "flux_z")) if k else "-"
print(f"{sys.argv[1]:10s} fp64 {d['value']/1e6:7.1f}M  fp32 {d['fp32']['value']/1e6:7.1f}M  flux64 {f(k)} flux32 {f(k32)} recon {k['recon']:.2f} frac {d['roofline']['frac']:.3f}")
PY
  done
done
