"""Check the paper's statements about the compressible TGV Mach sweep (Fig. "tg-vortex-
compressible", 256^3, Re 1600) on the output of tools/tgv_budget.py:

  1. Ma = 0.75 and 1.0 show regions of increasing kinetic energy (the paper: during 2 <= t <= 4),
     while the low-Mach cases decline monotonically;
  2. the peak of the total viscous dissipation eps_com = eps_s + eps_d is delayed and flattened as
     the Mach number increases;
  3. the Ma = 0.25 peak matches the Ma = 0.1 peak closely;
  4. for Ma >= 0.75 eps_com is higher than the near-incompressible case late in the run (t >= 11).

These are the paper's qualitative findings (figures only, SURVEY O-P16), so this is a check of the
trends, not parity.  usage: python tools/tgv_mach_trends.py budget.json
"""
import json
import sys

import numpy as np


def main(path):
    d = json.load(open(path))
    runs = {float(k): v for k, v in d["runs"].items()}
    out = {}
    for ma, r in sorted(runs.items()):
        t = np.array(r["t"])
        ek = np.array(r["E_k"])
        eps = np.array(r["eps_s"]) + np.array(r["eps_d"])
        dek = np.diff(ek)
        i = int(np.argmax(eps))
        out[ma] = dict(t=t, ek=ek, eps=eps, increasing_2_4=bool(np.any(dek[(t[1:] >= 2) & (t[1:] <= 4)] > 0)),
                       monotone=bool(np.all(dek <= 0)), t_peak=float(t[i]), peak=float(eps[i]))
        print(f"Ma {ma:4.2f}: E_k rises in 2<=t<=4: {out[ma]['increasing_2_4']!s:5}  monotone decline: "
              f"{out[ma]['monotone']!s:5}  peak eps_com {out[ma]['peak']:.5f} at t = {out[ma]['t_peak']:.1f}")
    res = {}
    hi = [m for m in out if m >= 0.75]
    lo = [m for m in out if m <= 0.25]
    res["1_rise_high_Ma"] = all(out[m]["increasing_2_4"] for m in hi) and all(out[m]["monotone"] for m in lo)
    ms = sorted(out)
    res["2_delay_and_flatten"] = out[ms[-1]]["t_peak"] > out[ms[0]]["t_peak"] and out[ms[-1]]["peak"] < out[ms[0]]["peak"]
    if 0.1 in out and 0.25 in out:
        res["3_ma025_matches_ma01"] = abs(out[0.25]["peak"] / out[0.1]["peak"] - 1) < 0.05
    if 0.1 in out and out[0.1]["t"][-1] >= 11:
        late = out[0.1]["t"] >= 11
        res["4_late_dissipation_higher"] = all(
            np.mean(out[m]["eps"][out[m]["t"] >= 11]) > np.mean(out[0.1]["eps"][late]) for m in hi)
    print(json.dumps(res))
    return res


if __name__ == "__main__":
    main(sys.argv[1])
