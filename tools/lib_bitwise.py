"""Run a fixed case (TGV n^3, CFL steps, fp32 and fp64) with the library HGKS_LIB points to and save the
states, so two builds can be compared bitwise.  usage: HGKS_LIB=... python tools/lib_bitwise.py out.npz [n] [steps]"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_01173_b200 import hgks as H  # noqa: E402
from paper_2207_01173_b200 import inputs  # noqa: E402

out = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 48
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
q, _ = inputs.tgv(n)
res = {}
for name, prec in (("fp64", H.HGKS_FP64), ("fp32", H.HGKS_FP32)):
    with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=inputs.tgv_params()["mu"], cfl=0.4, precision=prec,
                  device=0) as s:
        s.set_state(q)
        s.step(steps)
        res[name] = s.get_state()
np.savez(out, **res)
if len(sys.argv) > 4:
    ref = np.load(sys.argv[4])
    for k in res:
        print(k, "bitwise equal" if np.array_equal(ref[k], res[k]) else f"DIFFERS max {np.abs(ref[k] - res[k]).max():.3e}")
