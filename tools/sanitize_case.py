"""Small cases for compute-sanitizer (tools/gpu_sanitize.sh): TGV 32^3 fp64 + fp32, 2 steps (CUDA graph
path) + 1 step (plain path) with the per-step history on, and a 2-rank loopback group (halo copies,
reductions), a ragged channel grid (walls, tanh mesh, power-law mu, Pr fix: ragged flux tiles, the single-line
copy fallback) and the one-member NCCL communicator.  usage: python tools/sanitize_case.py
[single|loopback|ragged|nccl]"""
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
            # asynchronous host I/O: upload / commit / step / download overlapping, io_wait
            out = np.zeros_like(q)
            s.upload_state(q)
            s.commit_state()
            s.upload_state(q)
            s.step(1)
            s.download_state(out)
            s.commit_state()
            s.io_wait()
    print("single ok")
elif mode == "ragged":
    grid = (21, 18, 23)
    qr, _ = inputs.perturbed(grid, seed=3, amp=0.05)
    for prec in (H.HGKS_FP64, H.HGKS_FP32):
        with H.Solver(grid, (0.0, -1.0, 0.0), (2.0, 1.0, 1.0), mu=1e-3, mu_law=H.HGKS_MU_POWER, T_ref=1.0, omega=0.7,
                      prandtl=0.7, T_wall=1.0, bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                      stretch=(H.HGKS_UNIFORM, H.HGKS_TANH, H.HGKS_UNIFORM), stretch_b=(0.0, 2.0, 0.0),
                      force_mode=H.HGKS_FORCE_BULK, force=0.0, force_target=0.0, cfl=0.4, precision=prec) as s:
            s.set_state(qr)
            s.step(2)
            s.get_state()
    print("ragged ok")
elif mode == "nccl":
    with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=mu, cfl=0.4, nccl_id=H.hgks_get_nccl_id()) as s:
        s.set_state(q)
        s.step(2)
        s.diagnostics()
        s.get_state()
    print("nccl ok")
else:
    def work(rank, nranks, key):
        with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=mu, cfl=0.4, rank=rank, nranks=nranks,
                      group_key=key) as s:
            s.set_state(np.ascontiguousarray(q[:, s.z0:s.z0 + s.nz_local]))
            s.step(2)
            s.diagnostics()
            return s.get_state().shape
    print("loopback ok", H.run_loopback_group(2, work))
