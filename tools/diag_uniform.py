import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs
n = (16, 12, 10)
q = inputs.uniform(n, rho=1.2, vel=(0.3, -0.7, 0.45), p=0.9)
with H.Solver(n, (0, 0, 0), (1.6, 1.2, 1.0), mu=1e-3, dt_fixed=0.01) as s:
    s.set_state(q)
    L, dL = H.hgks_test_operator(s.ctx, 0.01, q.shape)
    for d in range(3):
        F = H.hgks_test_face_flux(s.ctx, d, n)
        for c in range(10):
            u, cnt = np.unique(F[c], return_counts=True)
            if len(u) > 1:
                print("dir", d, "comp", c, "distinct", len(u), "values", u[:4], "counts", cnt[:4])
                where = np.argwhere(F[c] != u[np.argmax(cnt)])
                print("    odd faces (z,y,x):", where[:8].tolist())
