"""Static FP64-pipe instruction count per source line of one flux kernel instance.
usage: python tools/sass_lines.py [mangled_substring] [topn]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

sub = sys.argv[1] if len(sys.argv) > 1 else "flux_kernelIdLi0ELi1ELb0"
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath("paper_2207_01173_b200/libhgks.so")], cwd=tmp, capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
parts = re.split(r"\n\s*\.text\.(\S+):", txt)
for i in range(1, len(parts), 2):
    if sub not in parts[i]:
        continue
    cur, cnt = None, collections.Counter()
    for l in parts[i + 1].splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", l)
        if m and m.group(1) in ("DFMA", "DMUL", "DADD"):
            cnt[cur] += 1
    print("total", sum(cnt.values()))
    src = {}
    for (f, ln), v in sorted(cnt.items(), key=lambda x: -x[1])[:topn]:
        if f not in src:
            p = [os.path.join("paper_2207_01173_b200/csrc", f)]
            src[f] = open(p[0]).read().splitlines() if os.path.exists(p[0]) else []
        text = src[f][ln - 1].strip()[:90] if ln <= len(src[f]) else ""
        print(f"{v:4d}  {f}:{ln}  {text}")
    break
