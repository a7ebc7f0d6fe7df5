"""Channel wall statistics from time-sampled x-z plane means.

The device reduction is hgks_plane_stats (one block per y plane, fixed order, NCCL sum over slabs);
this module only time-averages its [ny][16] outputs and forms the paper's normalised profiles.
Definitions (reading O-28):

  <.>          mean over the samples and the x and z directions
  phi'         phi - <phi>;  phi_rms = sqrt(<phi^2> - <phi>^2)
  tau_w        mu_w d<U>/dy at the wall: the quadratic through (0, 0) and the first two cell
               centres (exact for the laminar parabola), averaged over both walls
  rho_w        <p> of the wall-adjacent cells / T_w (isothermal wall, dp/dy = 0 at the wall)
  u_tau        sqrt(tau_w / rho_w), delta_nu = mu_w / (rho_w u_tau), y+ = s / delta_nu, s = wall distance
  <U>+         <U> / u_tau ; the Van Driest velocity (Eq. 10)
               <U>_VD+ = int_0^{<U>+} (<rho>/rho_w)^{1/2} d<U>+  (trapezoid from the wall)
  rms+         U_rms / u_tau, V_rms / u_tau, W_rms / u_tau
  -<rho U'V'>/<tau_w>  with <rho U'V'> = <rho U V> - <U><rho V> - <V><rho U> + <rho><U><V>
               (P:1227-1228); the upper half is mirrored (V changes sign)
  M_rms        sqrt(<M^2> - <M>^2), M = |U|/c ;  M_t = q / <c>, q^2 = <U'^2 + V'^2 + W'^2>

Profiles are folded onto the lower half (distance s from the nearer wall).
"""
from __future__ import annotations

import numpy as np

STAT_NAMES = ("rho", "U", "V", "W", "UU", "VV", "WW", "UV", "rhoU", "rhoV", "rhoUV", "c", "M", "MM", "T", "p")
_S = {k: i for i, k in enumerate(STAT_NAMES)}


class ChannelStats:
    """Accumulate plane means (hgks_plane_stats samples) and evaluate the wall statistics.

    y_centres: the ny cell-centre coordinates; walls at y_lo, y_hi (the channel's -H, H)."""

    def __init__(self, y_centres, mu_w: float, T_w: float, y_lo: float = -1.0, y_hi: float = 1.0):
        self.y = np.asarray(y_centres, dtype=np.float64)
        self.mu_w, self.T_w = float(mu_w), float(T_w)
        self.y_lo, self.y_hi = float(y_lo), float(y_hi)
        self.sum = np.zeros((self.y.size, len(STAT_NAMES)))
        self.samples = 0

    def add(self, plane_means: np.ndarray) -> None:
        pm = np.asarray(plane_means, dtype=np.float64)
        if pm.shape != self.sum.shape:
            raise ValueError(f"plane means of shape {pm.shape}, expected {self.sum.shape}")
        self.sum += pm
        self.samples += 1

    def mean(self) -> np.ndarray:
        if self.samples == 0:
            raise ValueError("no samples")
        return self.sum / self.samples

    @staticmethod
    def _wall_slope(s0, s1, u0, u1):
        # derivative at s = 0 of the quadratic through (0, 0), (s0, u0), (s1, u1)
        return (u0 * s1 * s1 - u1 * s0 * s0) / (s0 * s1 * (s1 - s0))

    def profiles(self) -> dict:
        m = self.mean()
        ny = self.y.size
        half = ny // 2
        lo = np.arange(half)                # lower half, wall distance increasing
        hi = ny - 1 - np.arange(half)       # upper half mirrored onto the lower one
        s_lo = self.y[lo] - self.y_lo
        s_hi = self.y_hi - self.y[hi]
        col = lambda k: m[:, _S[k]]
        U = col("U")
        dudy = 0.5 * (self._wall_slope(s_lo[0], s_lo[1], U[lo[0]], U[lo[1]]) +
                      self._wall_slope(s_hi[0], s_hi[1], U[hi[0]], U[hi[1]]))
        tau_w = self.mu_w * dudy
        rho_w = 0.5 * (col("p")[lo[0]] + col("p")[hi[0]]) / self.T_w
        u_tau = np.sqrt(tau_w / rho_w)
        delta_nu = self.mu_w / (rho_w * u_tau)

        def fold(v, odd=False):
            return 0.5 * (v[lo] + (-v[hi] if odd else v[hi]))

        var = {k: col(k + k) - col(k) ** 2 for k in ("U", "V", "W")}
        ruv = col("rhoUV") - col("U") * col("rhoV") - col("V") * col("rhoU") + col("rho") * col("U") * col("V")
        s = 0.5 * (s_lo + s_hi)
        Up = fold(U) / u_tau
        rho = fold(col("rho"))
        # Van Driest (Eq. 10): trapezoid of sqrt(<rho>/rho_w) dU+ from the wall (U+ = 0, rho = rho_w)
        w = np.sqrt(np.concatenate([[1.0], rho / rho_w]))
        dU = np.diff(np.concatenate([[0.0], Up]))
        U_vd = np.cumsum(0.5 * (w[1:] + w[:-1]) * dU)
        q2 = var["U"] + var["V"] + var["W"]
        return dict(
            s=s, y_plus=s / delta_nu, U_plus=Up, U_vd_plus=U_vd,
            u_rms_plus=np.sqrt(np.maximum(fold(var["U"]), 0.0)) / u_tau,
            v_rms_plus=np.sqrt(np.maximum(fold(var["V"]), 0.0)) / u_tau,
            w_rms_plus=np.sqrt(np.maximum(fold(var["W"]), 0.0)) / u_tau,
            reynolds_stress=-fold(ruv, odd=True) / tau_w,
            M_rms=np.sqrt(np.maximum(fold(col("MM") - col("M") ** 2), 0.0)),
            M_t=np.sqrt(np.maximum(fold(q2), 0.0)) / fold(col("c")),
            tau_w=tau_w, rho_w=rho_w, u_tau=u_tau, Re_tau=(self.y_hi - self.y_lo) / 2 / delta_nu,
            samples=self.samples,
        )
