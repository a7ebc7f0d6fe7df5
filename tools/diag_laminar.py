"""Trace the bulk controller on the laminar channel around a t_end-clamped step (debug helper)."""
import math
import numpy as np
from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs

ny, mu, Ma, rho_b, U_b = 32, 0.1, 0.05, 1.0, 1.0
Tw = 1.0 / (1.4 * Ma * Ma)
n = (5, ny, 5)
shape = n[::-1]
q = inputs.prim_to_cons(np.full(shape, rho_b), np.full(shape, U_b), 0.0, 0.0, rho_b * Tw)
with H.Solver(n, (0, -1, 0), (2 * math.pi, 1, math.pi), mu=mu, prandtl=0.7, T_wall=Tw,
              bc=(0, 1, 0), force_mode=H.HGKS_FORCE_BULK, force=0.0, force_target=1.0) as s:
    s.set_state(q)
    s.step(4000)
    for t_end in (5.0 + 1e-4, 5.0 + 1e-4 + 3e-7, 5.01, 5.02):
        dt = s.step(100000, t_end=t_end)
        f, m, rb = H.hgks_get_forcing(s.ctx)
        print(f"t={s.t:.9f} dt_last={dt:.3e} f/(3mu)={f/(3*mu):.6f} m-1={m-1:.3e}")
    for k in range(3):
        dt = s.step(1)
        f, m, rb = H.hgks_get_forcing(s.ctx)
        print(f"t={s.t:.9f} dt_last={dt:.3e} f/(3mu)={f/(3*mu):.6f} m-1={m-1:.3e}")
