"""Independent velocity-space quadrature for pinning the oracle's kinetic machinery.

This is a brute-force route to the same integrals the oracle evaluates with moment
recursions: it samples the Maxwellian g = rho (lam/pi)^{(K+3)/2} exp(-lam(|u-U|^2 + xi^2))
 on tensor quadrature grids and sums.  K = 2 (gamma = 1.4) is handled exactly:
the two internal degrees of freedom enter only through s = xi^2, whose density is
lam * exp(-lam s) on s > 0, integrated by Gauss-Laguerre.

  * u: Gauss-Hermite (full space) or Gauss-Legendre on a truncated half line (u>0 / u<0)
  * v, w: Gauss-Hermite
  * s = xi^2: Gauss-Laguerre (exact for polynomials in s of degree < 2*NS)

It shares nothing with oracle/hgks_oracle.c (no recursion, no erfc, no closed-form solve).
"""
from __future__ import annotations

import math

import numpy as np

NH = 18   # Gauss-Hermite nodes per velocity axis: exact to polynomial degree 35
NS = 8    # Gauss-Laguerre nodes for s = xi^2
NL = 160  # Gauss-Legendre nodes on the truncated half line


def _gh(lam, U, n=NH):
    x, w = np.polynomial.hermite.hermgauss(n)
    return U + x / math.sqrt(lam), w / math.sqrt(math.pi)


def _half(lam, U, sign, n=NL):
    """nodes/weights of sqrt(lam/pi) exp(-lam (u-U)^2) on u*sign > 0 (sign=+1: u>0)."""
    sig = 1.0 / math.sqrt(2 * lam)
    if sign > 0:
        a, b = 0.0, max(0.0, U + 40 * sig)
    else:
        a, b = min(0.0, U - 40 * sig), 0.0
    if b - a <= 0:
        return np.zeros(1), np.zeros(1)
    x, w = np.polynomial.legendre.leggauss(n)
    # split the interval in 8 panels for accuracy on long intervals
    nodes, weights = [], []
    edges = np.linspace(a, b, 9)
    for lo, hi in zip(edges[:-1], edges[1:]):
        u = 0.5 * (hi - lo) * x + 0.5 * (hi + lo)
        nodes.append(u)
        weights.append(0.5 * (hi - lo) * w * math.sqrt(lam / math.pi) * np.exp(-lam * (u - U) ** 2))
    return np.concatenate(nodes), np.concatenate(weights)


def grid(mx, which=0):
    """Quadrature points (u, v, w, s) and weights of g/rho for Maxwellian mx=(rho,U,V,W,lam), K=2.
    which: 0 full, +1 u>0, -1 u<0."""
    rho, U, V, W, lam = mx
    if which == 0:
        u, wu = _gh(lam, U)
    else:
        u, wu = _half(lam, U, which)
    v, wv = _gh(lam, V)
    w, ww = _gh(lam, W)
    xs, ws = np.polynomial.laguerre.laggauss(NS)
    s = xs / lam  # int lam e^{-lam s} f(s) ds = sum ws f(xs/lam)
    U_, V_, W_, S_ = np.meshgrid(u, v, w, s, indexing="ij")
    wt = (wu[:, None, None, None] * wv[None, :, None, None] * ww[None, None, :, None]
          * ws[None, None, None, :])
    return U_.ravel(), V_.ravel(), W_.ravel(), S_.ravel(), wt.ravel()


def psi(u, v, w, s):
    return np.stack([np.ones_like(u), u, v, w, 0.5 * (u * u + v * v + w * w + s)])


def poly(al, u, v, w, s):
    """alpha . psi"""
    return al[0] + al[1] * u + al[2] * v + al[3] * w + 0.5 * al[4] * (u * u + v * v + w * w + s)


def moment(mx, fun, which=0):
    """int fun(u,v,w,s) g/rho dXi  (fun returns (..., npts))."""
    u, v, w, s, wt = grid(mx, which)
    return fun(u, v, w, s) @ wt


def maxwellian_of(Q, K=2.0):
    """Maxwellian parameters of conservative Q by DEFINITION: U = m/rho and lam such that the
    energy moment matches; verified against quadrature in the tests."""
    rho = Q[0]
    U, V, W = Q[1] / rho, Q[2] / rho, Q[3] / rho
    e = Q[4] / rho - 0.5 * (U * U + V * V + W * W)  # = (K+3)/(4 lam)
    return np.array([rho, U, V, W, (K + 3) / (4 * e)])


def moment_matrix(mx):
    """M[k, n] = <psi_n psi_k>/rho by quadrature."""
    u, v, w, s, wt = grid(mx, 0)
    P = psi(u, v, w, s)
    return (P * wt) @ P.T


def slopes(mx, dW):
    """a_i solving <a_i . psi psi> = dW_i / rho, and A solving <(u a1 + v a2 + w a3 + A) psi> = 0,
    all by quadrature-assembled matrices and numpy.linalg.solve."""
    M = moment_matrix(mx)
    a = [np.linalg.solve(M, np.asarray(dW[i]) / mx[0]) for i in range(3)]
    u, v, w, s, wt = grid(mx, 0)
    P = psi(u, v, w, s)
    rhs = -((u * poly(a[0], u, v, w, s) + v * poly(a[1], u, v, w, s) + w * poly(a[2], u, v, w, s)) * P) @ wt
    A = np.linalg.solve(M, rhs)
    return a, A
