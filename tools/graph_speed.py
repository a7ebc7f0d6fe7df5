"""Steps per second with and without the CUDA-graph replay of step pairs (small TGV grids)."""
import math
import os
import subprocess
import sys

code = r"""
import math, sys, time, torch
sys.path.insert(0, '.')
from paper_2207_01173_b200 import hgks as H, inputs
n = int(sys.argv[1])
q, _ = inputs.tgv(n)
with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=1 / 1600, cfl=0.4) as s:
    s.set_state(torch.from_numpy(q).cuda())
    s.step(10)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.step(200)
    dt = time.perf_counter() - t0
print(f"{n} {200 / dt:.1f} steps/s {n ** 3 * 200 / dt / 1e6:.1f} M cell-updates/s")
"""
for n in (32, 64, 128):
    for g in ("1", "0"):
        env = dict(os.environ, HGKS_GRAPHS=g)
        r = subprocess.run([sys.executable, "-c", code, str(n)], env=env, capture_output=True, text=True)
        print(f"graphs={g}", (r.stdout or r.stderr).strip().splitlines()[-1])
