"""Per-source-line FP64 instruction counts (DFMA/DMUL/DADD/other D*) of one kernel in an ncu report.
usage: ncu_fp64_lines.py report.ncu-rep lib.so kernel_substring mangled_substring [topn]"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(__file__))
import ncu_lines as N  # noqa: E402


def main(rep, lib, ksub, msub, topn=40):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    amap = N.sass_lines(cubin, msub)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', txt)[1:]
    b = [b for b in blocks if ksub in b.splitlines()[0]][0]
    rows = list(csv.reader(b.splitlines()[1:]))
    hdr = rows[0]
    by = defaultdict(lambda: defaultdict(int))
    tot = defaultdict(int)
    base = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        try:
            addr = int(d["Address"], 16)
        except Exception:
            continue
        if base is None:
            base = addr
        src, _ = amap.get(addr - base, (None, ""))
        op = re.sub(r"^@!?U?P\w+\s+", "", d.get("Source", "").strip()).split(" ")[0].split(".")[0]
        n = int(float(d["Instructions Executed"] or 0))
        by[src][op] += n
        tot[op] += n
    fp = ("DFMA", "DMUL", "DADD")
    lines = sorted(by.items(), key=lambda kv: -sum(kv[1][o] for o in fp))
    warps = tot["DFMA"] + tot["DMUL"] + tot["DADD"]
    print("FP64 warp-inst total", warps, {o: tot[o] for o in fp})
    for src, ops in lines[:topn]:
        f = sum(ops[o] for o in fp)
        print(f"{100 * f / warps:6.2f}%  {f:>11d}  DFMA {ops['DFMA']:>10d} DMUL {ops['DMUL']:>10d} DADD {ops['DADD']:>9d}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5]) if len(sys.argv) > 5 else 40)
