"""Build a libhgks variant with ptxas -v and print registers / spills per flux kernel.
usage: python tools/ptxas_summary.py [-DNAME=VAL ...] [-out=libname.so]"""
import re
import subprocess
import sys

out = subprocess.run([sys.executable, "paper_2207_01173_b200/build.py", "-v", *sys.argv[1:]], capture_output=True,
                     text=True)
txt = out.stdout + out.stderr
cur = None
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur and ("spill" in line or "Used" in line):
        if "flux_kernel" in cur or "recon" in cur:
            dm = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
            dm = re.sub(r"\(.*", "", dm)
            print(f"{dm:60s} {line.strip()}")
print(txt.splitlines()[-1])
