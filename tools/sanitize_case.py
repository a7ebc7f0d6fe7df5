"""Small cases for compute-sanitizer (tools/gpu_sanitize.sh): TGV 32^3 fp64 + fp32, 2 steps (CUDA graph
path) + 1 step (plain path) with the per-step history on, and a 2-rank loopback group (halo copies,
reductions).  usage: python tools/sanitize_case.py [single|loopback]"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_2207_01173_b200 import hgks as H  # noqa: E402
from paper_2207_01173_b200 import inputs  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "single"
n = 32
q, _ = inputs.tgv(n)
mu = inputs.tgv_params()["mu"]
if mode == "single":
    for prec in (H.HGKS_FP64, H.HGKS_FP32):
        with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=mu, cfl=0.4, precision=prec) as s:
            H.hgks_history_enable(s.ctx, 8)
            s.set_state(q)
            s.step(2)
            s.step(1)
            H.hgks_history_read(s.ctx, 8)
            s.diagnostics()
            s.get_state()
    print("single ok")
else:
    def work(rank, nranks, key):
        with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=mu, cfl=0.4, rank=rank, nranks=nranks,
                      group_key=key) as s:
            s.set_state(np.ascontiguousarray(q[:, s.z0:s.z0 + s.nz_local]))
            s.step(2)
            s.diagnostics()
            return s.get_state().shape
    print("loopback ok", H.run_loopback_group(2, work))
