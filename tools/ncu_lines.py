"""Attribute ncu per-instruction samples of one kernel to CUDA source lines (via nvdisasm -g).
usage: ncu_lines.py report.ncu-rep lib.so kernel_substring [kernel_index]"""
import csv
import re
import subprocess
import sys
import tempfile
import os
from collections import defaultdict


def sass_lines(cubin, mangled_sub):
    out = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
    fn = None
    cur = None
    amap = {}
    for l in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            fn = m.group(1)
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m and fn and mangled_sub in fn:
            amap[int(m.group(1), 16)] = (cur, m.group(2).split(";")[0].strip())
    return amap


def main(rep, lib, ksub, kidx=0, mangled_sub=None):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    # split per kernel blocks
    blocks = re.split(r'(?m)^"Kernel Name",', txt)[1:]
    sel = [b for b in blocks if ksub in b.splitlines()[0]]
    b = sel[kidx]
    lines = b.splitlines()
    rows = list(csv.reader(lines[1:]))
    hdr = rows[0]
    amap = sass_lines(cubin, mangled_sub or "flux_kernel")
    by_line = defaultdict(lambda: [0, 0])
    by_op = defaultdict(lambda: [0, 0])
    tot = 0
    base = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        try:
            addr = int(d["Address"], 16)
        except Exception:
            continue
        if base is None:
            base = addr
        addr -= base
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        ins = int(float(d["Instructions Executed"] or 0))
        tot += s
        src, op = amap.get(addr, (None, d.get("Source", "")))
        by_line[src][0] += s
        by_line[src][1] += ins
        opc = re.sub(r"^@!?U?P\w+\s+", "", d.get("Source", "").strip()).split(" ")[0].split(".")[0]
        by_op[opc][0] += s
        by_op[opc][1] += ins
    print("total samples", tot)
    for k, v in sorted(by_line.items(), key=lambda x: -x[1][0])[:int(__import__("os").environ.get("TOPN","45"))]:
        print(f"{v[0] / tot * 100:6.2f}%  inst={v[1]:>12d}  {k}")
    print("-- by opcode")
    for k, v in sorted(by_op.items(), key=lambda x: -x[1][0])[:20]:
        print(f"{v[0] / tot * 100:6.2f}%  inst={v[1]:>12d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 0,
         sys.argv[5] if len(sys.argv) > 5 else None)
