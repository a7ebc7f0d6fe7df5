"""FP32-vs-FP64 twin run (SURVEY §8(f) NEXT-3 study; the paper's FP32/FP64 comparison).

Runs the TGV (Re 1600, Ma 0.1) from the same initial field in both precisions on one GPU and records,
at fixed output times, the on-device volume diagnostics (E_k, enstrophy, eps_s, eps_d; NEXT-2) of both
runs and the normwise state difference (O-19) between them.  Output: one JSON document.

usage: python tools/precision_twin.py [--n 128] [--t-end 10] [--every 0.25] [--out file.json]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_01173_b200 import hgks as H  # noqa: E402
from paper_2207_01173_b200 import inputs  # noqa: E402


def normwise(a, b):
    mom = np.sqrt(b[1] ** 2 + b[2] ** 2 + b[3] ** 2).max()
    den = [np.abs(b[0]).max(), mom, mom, mom, np.abs(b[4]).max()]
    return [float(np.abs(a[v] - b[v]).max() / den[v]) for v in range(5)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--t-end", type=float, default=10.0)
    ap.add_argument("--every", type=float, default=0.25)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    n = a.n
    q, _ = inputs.tgv(n)
    prm = inputs.tgv_params()
    solvers = {p: H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=prm["mu"], cfl=0.4, precision=c)
               for p, c in (("fp64", H.HGKS_FP64), ("fp32", H.HGKS_FP32))}
    for s in solvers.values():
        s.set_state(q)
    rec = {"config": {"workload": f"tgv{n}", "re": prm["re"], "ma": prm["ma"], "cfl": 0.4, "t_end": a.t_end,
                      "every": a.every}, "t": [], "fp64": {k: [] for k in H.DIAG_NAMES},
           "fp32": {k: [] for k in H.DIAG_NAMES}, "state_diff": [], "steps": {"fp64": 0, "fp32": 0}, "wall_s": {}}
    wall = {"fp64": 0.0, "fp32": 0.0}
    t = 0.0
    k = 0
    while t < a.t_end - 1e-12:
        t_next = min(a.t_end, (k + 1) * a.every)
        for p, s in solvers.items():
            t0 = time.perf_counter()
            while s.t < t_next * (1 - 1e-13):
                s.step(100000, t_end=t_next)
            wall[p] += time.perf_counter() - t0
            d = H.hgks_diagnostics(s.ctx)
            for name, v in zip(H.DIAG_NAMES, d):
                rec[p][name].append(float(v))
        t = t_next
        k += 1
        rec["t"].append(t)
        q64, q32 = solvers["fp64"].get_state(), solvers["fp32"].get_state()
        rec["state_diff"].append(normwise(q32, q64))
        print(f"t={t:6.3f} Ek64={rec['fp64']['E_k'][-1]:.6e} Ek32={rec['fp32']['E_k'][-1]:.6e} "
              f"zeta64={rec['fp64']['enstrophy'][-1]:.5e} zeta32={rec['fp32']['enstrophy'][-1]:.5e} "
              f"diff={max(rec['state_diff'][-1]):.2e}", flush=True)
    for s in solvers.values():
        s.close()
    e64, e32 = np.array(rec["fp64"]["E_k"]), np.array(rec["fp32"]["E_k"])
    z64, z32 = np.array(rec["fp64"]["enstrophy"]), np.array(rec["fp32"]["enstrophy"])
    rec["wall_s"] = wall
    rec["summary"] = {
        "max_rel_diff_E_k": float(np.max(np.abs(e32 - e64) / e64)),
        "max_rel_diff_enstrophy": float(np.max(np.abs(z32 - z64) / z64)),
        "t_enstrophy_peak_fp64": float(rec["t"][int(np.argmax(z64))]),
        "t_enstrophy_peak_fp32": float(rec["t"][int(np.argmax(z32))]),
        "max_state_diff": float(np.max(rec["state_diff"])),
    }
    print(json.dumps(rec["summary"]))
    if a.out:
        json.dump(rec, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
