"""Per-source-line stall breakdown of one kernel in an ncu report (via nvdisasm -g line map).
usage: ncu_line_stalls.py report.ncu-rep lib.so 'kernel name substring' mangled_substring [topn]"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import sass_lines  # noqa: E402

rep, lib, ksub, msub = sys.argv[1:5]
topn = int(sys.argv[5]) if len(sys.argv) > 5 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
blocks = re.split(r'(?m)^"Kernel Name",', txt)[1:]
b = [b for b in blocks if ksub in b.splitlines()[0]][0]
rows = list(csv.reader(b.splitlines()[1:]))
hdr = rows[0]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
amap = sass_lines(cubin, msub)
agg = defaultdict(lambda: defaultdict(float))
tot = 0
base = None
for r in rows[1:]:
    d = dict(zip(hdr, r))
    try:
        addr = int(d["Address"], 16)
    except Exception:
        continue
    base = addr if base is None else base
    src = amap.get(addr - base, (None, ""))[0]
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    tot += s
    agg[src]["all"] += s
    for h in stalls:
        agg[src][h] += float(d[h] or 0)
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1]["all"])[:topn]:
    top = sorted(((h[6:], v[h]) for h in stalls), key=lambda x: -x[1])[:4]
    print(f"{v['all'] / tot * 100:6.2f}%  {str(k):36s} " + " ".join(f"{n}={x / v['all'] * 100:.0f}%" for n, x in top if x > 0))
