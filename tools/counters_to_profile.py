"""Turn the ncu counter CSVs of tools/gpu_counters_round.sh into profiles/ summaries.

usage: python tools/counters_to_profile.py TAG N   (N = grid n of the profiled run, 256)
Writes profiles/flux_flops.json (read by bench.py for roofline.achieved / traffic) and
profiles/<TAG>_kernel_counters.md (human-readable table)."""
import csv
import io
import json
import sys
from collections import defaultdict


def load(path):
    txt = open(path).read()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    launches = defaultdict(dict)
    names = {}
    for r in rows:
        launches[int(r["ID"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        names[int(r["ID"])] = r["Kernel Name"]
    return [(names[i], launches[i]) for i in sorted(launches)]


def faces(kname, n):
    # flux_kernel<T, DIR, STAGE>: (n+1) n^2 faces; recon/update: per face-line / per cell
    return (n + 1) * n * n


def main(tag, n):
    out = {"source": f"ncu SASS counters (tools/gpu_counters_round.sh {tag}), TGV {n}^3", "grid": n}
    md = [f"# Kernel counters, round tag `{tag}` (TGV {n}^3, one step, ncu --clock-control none)\n",
          "| precision | kernel | time ms | FP64 flop (DFMA*2+DMUL+DADD) | FP32 flop | flop/face | FP64 pipe % | DRAM read MB | DRAM write MB |",
          "|---|---|---|---|---|---|---|---|---|"]
    for prec, path in (("fp64", f"gpurun_out/counters64_{tag}.csv"), ("fp32", f"gpurun_out/counters32_{tag}.csv")):
        per = defaultdict(list)
        for name, m in load(path):
            f64 = 2 * m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0) + \
                m.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0) + \
                m.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
            f32 = 2 * m.get("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", 0) + \
                m.get("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", 0) + \
                m.get("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", 0)
            short = name.split("(")[0].replace("void ", "")
            t = m["gpu__time_duration.sum"] * 1e-6
            fl = f64 if prec == "fp64" else f32
            per[short].append(dict(ms=t, flop=fl, dram=m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]))
            md.append(f"| {prec} | `{short}` | {t:.3f} | {f64:.4g} | {f32:.4g} | {fl / faces(short, n):.0f} | "
                      f"{m.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                      f"{m['dram__bytes_read.sum'] / 1e6:.0f} | {m['dram__bytes_write.sum'] / 1e6:.0f} |")
        for stage in (1, 2):
            # flux_kernel<T, DIR, STAGE[, PRF]>: the stage is the third template argument
            ks = [v for k, vs in per.items() if "flux_kernel" in k
                  and k.split("<", 1)[1].rstrip(">").split(",")[2].strip() == str(stage) for v in vs]
            if ks:
                flop = sum(v["flop"] for v in ks) / len(ks)
                out[f"{prec}_flop_per_face_stage{stage}"] = flop / faces("flux", n)
                out[f"{prec}_dram_bytes_per_launch_stage{stage}"] = sum(v["dram"] for v in ks) / len(ks)
    out["flop_per_face_stage1"] = out.get("fp64_flop_per_face_stage1")
    out["flop_per_face_stage2"] = out.get("fp64_flop_per_face_stage2")
    out["dram_bytes_per_launch"] = 0.5 * (out.get("fp64_dram_bytes_per_launch_stage1", 0) +
                                          out.get("fp64_dram_bytes_per_launch_stage2", 0))
    json.dump(out, open("profiles/flux_flops.json", "w"), indent=1)
    open(f"profiles/{tag}_kernel_counters.md", "w").write("\n".join(md) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
