"""Harness diagnostics applied identically to oracle and GPU outputs (fp64, numpy).

E_k and enstrophy (O-24), plus the normwise error metric O-19."""
import numpy as np


def kinetic_energy(q, rho0=1.0):
    """E_k = 1/(rho0 |Omega|) int 1/2 rho |U|^2 dOmega on a uniform grid."""
    return float(0.5 * ((q[1] ** 2 + q[2] ** 2 + q[3] ** 2) / q[0]).mean() / rho0)


def _d(f, axis, h):
    """4th-order central difference, periodic."""
    return (8 * (np.roll(f, -1, axis) - np.roll(f, 1, axis)) - (np.roll(f, -2, axis) - np.roll(f, 2, axis))) / (12 * h)


def enstrophy(q, dx, rho0=1.0):
    """zeta = 1/(rho0 |Omega|) int 1/2 rho |omega|^2 dOmega, omega = curl U (O-24)."""
    rho = q[0]
    U, V, W = q[1] / rho, q[2] / rho, q[3] / rho
    # arrays are [z][y][x]: axis 2 = x, 1 = y, 0 = z
    dx_, dy_, dz_ = dx
    wx = _d(W, 1, dy_) - _d(V, 0, dz_)
    wy = _d(U, 0, dz_) - _d(W, 2, dx_)
    wz = _d(V, 2, dx_) - _d(U, 1, dy_)
    return float((0.5 * rho * (wx * wx + wy * wy + wz * wz)).mean() / rho0)


def normwise_error(a, b):
    """O-19: per conservative variable max|a-b| / max|b|, momenta sharing max|rho U|."""
    a, b = np.asarray(a), np.asarray(b)
    mom = np.sqrt(b[1] ** 2 + b[2] ** 2 + b[3] ** 2).max()
    den = [np.abs(b[0]).max(), mom, mom, mom, np.abs(b[4]).max()]
    return np.array([np.abs(a[v] - b[v]).max() / den[v] for v in range(5)])
