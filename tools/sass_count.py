"""Static SASS instruction counts of the flux kernels in libhgks.so (FP64 pipe ops, LDS, spills).
usage: python tools/sass_count.py [lib.so]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

lib = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else "paper_2207_01173_b200/libhgks.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-c", cubin], capture_output=True, text=True).stdout
parts = re.split(r"\n\s*\.text\.(\S+):", txt)
for i in range(1, len(parts), 2):
    name, body = parts[i], parts[i + 1]
    m = re.search(r"flux_kernelI([df])Li(\d)ELi(\d)EL[bi](\d)", name)
    if not m:
        continue
    ops = collections.Counter()
    for l in body.splitlines():
        mm = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", l)
        if mm:
            ops[mm.group(1)] += 1
    fp = ops["DFMA"] + ops["DMUL"] + ops["DADD"] if m.group(1) == "d" else ops["FFMA"] + ops["FMUL"] + ops["FADD"]
    print(f"{m.group(1)} dir{m.group(2)} st{m.group(3)} prf{m.group(4)}: fp={fp:5d} (fma {ops['DFMA'] or ops['FFMA']}) "
          f"lds={ops['LDS']} ldl={ops['LDL']} stl={ops['STL']} total={sum(ops.values())}")
