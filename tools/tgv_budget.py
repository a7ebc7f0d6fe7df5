"""Compressible TGV Mach sweep and kinetic-energy budget closure.

For each Mach number the TGV (Re 1600, uniform temperature initial field) is advanced on
one GPU and the on-device diagnostics are recorded at fixed output times: E_k, the two terms of the
paper's dissipation rate eps_com = eps_s + eps_d and the pressure-dilatation Pi.  The
resolved budget is dE_k/dt = Pi - eps_s - eps_d; the residual
    r = -dE_k/dt - (eps_s + eps_d - Pi)
(dE_k/dt by central differences of the output series) is the scheme's numerical dissipation, which
shrinks with resolution.  Output: one JSON document (per Mach: t, E_k, eps_s, eps_d, Pi, residual).

usage: python tools/tgv_budget.py [--n 64] [--mach 0.1,0.25,0.5,1.0] [--t-end 10] [--every 0.1] [--out f]
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


def run(n, ma, t_end, every, precision):
    prm = inputs.tgv_params(ma=ma)
    q, _ = inputs.tgv(n, ma=ma)
    names = ("E_k", "eps_s", "eps_d", "p_dil", "enstrophy")
    rec = {"t": [], **{k: [] for k in names}, "steps": 0}
    t0 = time.perf_counter()
    with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=prm["mu"], cfl=0.4, precision=precision) as s:
        s.set_state(q)
        k = 0
        while True:
            d = s.diagnostics()
            rec["t"].append(s.t)
            for name in names:
                rec[name].append(float(d[name]))
            if s.t >= t_end * (1 - 1e-13):
                break
            k += 1
            s.step(1_000_000, t_end=min(t_end, k * every))
    rec["wall_s"] = time.perf_counter() - t0
    t = np.array(rec["t"])
    ek = np.array(rec["E_k"])
    diss = np.array(rec["eps_s"]) + np.array(rec["eps_d"]) - np.array(rec["p_dil"])
    dek = np.gradient(ek, t)
    rec["residual"] = (-dek - diss).tolist()  # numerical dissipation
    rec["summary"] = {
        "E_k_end": float(ek[-1]),
        "peak_eps_com": float(np.max(np.array(rec["eps_s"]) + np.array(rec["eps_d"]))),
        "t_peak_eps_com": float(t[int(np.argmax(np.array(rec["eps_s"]) + np.array(rec["eps_d"])))]),
        "max_abs_p_dil": float(np.max(np.abs(rec["p_dil"]))),
        "max_eps_d_over_eps_s": float(np.max(np.array(rec["eps_d"]) / np.maximum(rec["eps_s"], 1e-300))),
        # integrated over the run: numerical share of the total dissipation -dE_k/dt + Pi
        "numerical_share": float(np.trapezoid(np.array(rec["residual"]), t) / np.trapezoid(-dek + np.array(rec["p_dil"]), t)),
    }
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--mach", default="0.1,0.25,0.5,1.0")
    ap.add_argument("--t-end", type=float, default=10.0)
    ap.add_argument("--every", type=float, default=0.1)
    ap.add_argument("--fp32", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = {"config": {"workload": f"tgv{a.n}", "re": 1600, "t_end": a.t_end, "every": a.every,
                      "precision": "fp32" if a.fp32 else "fp64"}, "runs": {}}
    for ma in (float(x) for x in a.mach.split(",")):
        r = run(a.n, ma, a.t_end, a.every, H.HGKS_FP32 if a.fp32 else H.HGKS_FP64)
        out["runs"][str(ma)] = r
        print(f"Ma {ma}: {json.dumps(r['summary'])}  wall {r['wall_s']:.1f}s", flush=True)
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
