"""Per-region share of ncu stall samples and instructions of one kernel: each sampled source line is
attributed to the nearest preceding region marker (a function definition in gks_device.cuh, a
'// ---- phase' comment or kernel definition in hgks_kernels.cuh).
usage: ncu_regions.py report.ncu-rep lib.so "kernel name substring" mangled_substring [faces]"""
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(__file__))
from ncu_lines import main as _unused  # noqa: F401  (same directory helper)
import ncu_lines

SRC = {"gks_device.cuh": "paper_2207_01173_b200/csrc/gks_device.cuh",
       "hgks_kernels.cuh": "paper_2207_01173_b200/csrc/hgks_kernels.cuh"}


def markers(path):
    out = []
    for i, l in enumerate(open(path).read().splitlines(), 1):
        m = re.search(r"(?:HD|__device__ __forceinline__|__global__ void|__host__ __device__ __forceinline__)\s+(?:[\w:<>,\s\*&]+?\s)?(\w+)\s*\(", l)
        if m and not l.strip().startswith("//"):
            out.append((i, m.group(1)))
        m = re.search(r"// ---- (phase \w+)", l)
        if m:
            out.append((i, m.group(1)))
        m = re.search(r"\b(flux_kernel|recon_kernel|update_kernel)\(", l)
        if m and "__global__" not in l and "<<<" not in l:
            out.append((i, m.group(1)))
    return sorted(out)


def region(file, line, mk):
    best = "?"
    for l0, name in mk.get(file, []):
        if l0 <= line:
            best = name
    return f"{file.split('.')[0]}:{best}"


if __name__ == "__main__":
    rep, lib, ksub, mangled = sys.argv[1:5]
    faces = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
    mk = {k: markers(v) for k, v in SRC.items()}
    import io
    import contextlib
    buf = io.StringIO()
    os.environ["TOPN"] = "100000"
    with contextlib.redirect_stdout(buf):
        ncu_lines.main(rep, lib, ksub, 0, mangled)
    agg = {}
    for l in buf.getvalue().splitlines():
        m = re.match(r"\s*([\d.]+)%\s+inst=\s*(\d+)\s+\('(\S+)', (\d+)\)", l)
        if not m:
            continue
        r = region(m.group(3), int(m.group(4)), mk)
        a = agg.setdefault(r, [0.0, 0])
        a[0] += float(m.group(1))
        a[1] += int(m.group(2))
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{v[0]:6.2f}%  warp-inst/face {v[1] / faces:8.1f}  {k}")
