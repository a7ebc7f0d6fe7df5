"""Seeded, synthetic input generators shared by the tests, bench.py and smoke().

This module holds none of the method's arithmetic (no reconstruction, flux, time
integration or CFL): it only evaluates the paper's initial conditions and test-case
fields in fp64 with numpy, in the ABI layout [5][nz][ny][nx] (x fastest) of
conservative variables (rho, rhoU, rhoV, rhoW, rhoE).

Recipes (DESIGN.md §"Inputs"):
  * tgv         Taylor-Green vortex: periodic [-pi, pi]^3, cell-centre point
                values (O-14), uniform temperature so rho = p/p0 (O-15), Ma = 0.1
                (c0 = 10, p0 = rho0 c0^2/gamma), gamma = 1.4.
  * density_wave  rho = 1 + A sin(pi(k.x)), U = (1,1,1) or given, p = 1 on [0,2]^3, exact
                cell averages by 4-point Gauss-Legendre per axis (O-P4, O-14).
  * perturbed   a smooth random Fourier field around a uniform state (seeded), for
                parity tests that must exercise every branch of the flux.
"""
from __future__ import annotations

import math

import numpy as np

GAMMA = 1.4


def tgv_params(ma: float = 0.1, re: float = 1600.0, gamma: float = GAMMA):
    """TGV constants: L = V0 = rho0 = 1, c0 = V0/Ma, p0 = rho0 c0^2 / gamma, mu = 1/Re."""
    c0 = 1.0 / ma
    p0 = c0 * c0 / gamma
    return dict(gamma=gamma, p0=p0, mu=1.0 / re, c0=c0, ma=ma, re=re)


def cell_centres(n: int, lo: float, hi: float) -> np.ndarray:
    h = (hi - lo) / n
    return lo + (np.arange(n) + 0.5) * h


def prim_to_cons(rho, U, V, W, p, gamma=GAMMA) -> np.ndarray:
    rho, U, V, W, p = np.broadcast_arrays(rho, U, V, W, p)
    q = np.empty((5,) + rho.shape)
    q[0] = rho
    q[1] = rho * U
    q[2] = rho * V
    q[3] = rho * W
    q[4] = p / (gamma - 1.0) + 0.5 * rho * (U * U + V * V + W * W)
    return q


def tgv(n, ma: float = 0.1, gamma: float = GAMMA, z_begin: int = 0, nz_local: int | None = None):
    """TGV initial field on an n^3 (or (nx,ny,nz)) grid over [-pi,pi]^3.

    Returns (q [5][nz_local][ny][nx], dx tuple).  z_begin/nz_local select a slab (rank slab).
    """
    if isinstance(n, int):
        n = (n, n, n)
    nx, ny, nz = n
    if nz_local is None:
        nz_local = nz - z_begin
    prm = tgv_params(ma=ma, gamma=gamma)
    p0 = prm["p0"]
    x = cell_centres(nx, -math.pi, math.pi)
    y = cell_centres(ny, -math.pi, math.pi)
    z = cell_centres(nz, -math.pi, math.pi)[z_begin:z_begin + nz_local]
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    U = np.sin(X) * np.cos(Y) * np.cos(Z)
    V = -np.cos(X) * np.sin(Y) * np.cos(Z)
    W = np.zeros_like(U)
    p = p0 + (1.0 / 16.0) * (np.cos(2 * X) + np.cos(2 * Y)) * (np.cos(2 * Z) + 2.0)
    rho = p / p0
    dx = (2 * math.pi / nx, 2 * math.pi / ny, 2 * math.pi / nz)
    return np.ascontiguousarray(prim_to_cons(rho, U, V, W, p, gamma)), dx


def density_wave(n, amp: float = 0.2, k=(1, 1, 1), vel=(1.0, 1.0, 1.0), p: float = 1.0,
                 gamma: float = GAMMA, length: float = 2.0):
    """Exact cell averages of rho = 1 + amp sin(pi k.x), constant velocity and pressure on
    [0, length]^3 periodic (O-P4).  Returns (q, dx)."""
    if isinstance(n, int):
        n = (n, n, n)
    nx, ny, nz = n
    h = (length / nx, length / ny, length / nz)
    # 4-point Gauss-Legendre per axis: exact to degree 7 for the separable average of sin
    gx, gw = np.polynomial.legendre.leggauss(4)
    rho = np.zeros((nz, ny, nx))
    xc = [cell_centres(m, 0.0, length) for m in (nx, ny, nz)]
    for a, wa in zip(gx, gw):
        for b, wb in zip(gx, gw):
            for c, wc in zip(gx, gw):
                Z, Y, X = np.meshgrid(xc[2] + 0.5 * h[2] * c, xc[1] + 0.5 * h[1] * b,
                                      xc[0] + 0.5 * h[0] * a, indexing="ij")
                rho += (wa * wb * wc / 8.0) * (1.0 + amp * np.sin(math.pi * (k[0] * X + k[1] * Y + k[2] * Z)))
    q = np.empty((5, nz, ny, nx))
    q[0] = rho
    # rho*U averages to <rho> U for constant U; energy average: p/(g-1) + 0.5 <rho>|U|^2
    for d in range(3):
        q[1 + d] = rho * vel[d]
    q[4] = p / (gamma - 1.0) + 0.5 * rho * (vel[0] ** 2 + vel[1] ** 2 + vel[2] ** 2)
    return q, h


def uniform(n, rho=1.0, vel=(0.3, -0.2, 0.1), p=1.0, gamma: float = GAMMA):
    if isinstance(n, int):
        n = (n, n, n)
    nx, ny, nz = n
    q = prim_to_cons(np.full((nz, ny, nx), rho), vel[0], vel[1], vel[2], p, gamma)
    return np.ascontiguousarray(q)


def perturbed(n, seed: int = 0, amp: float = 0.05, modes: int = 3, base=(1.0, 0.2, -0.1, 0.15, 1.0),
              gamma: float = GAMMA, length: float = 2 * math.pi):
    """Smooth seeded random periodic field: each primitive = base * (1 + sum of `modes` random
    Fourier modes of relative amplitude amp).  Returns (q, dx)."""
    if isinstance(n, int):
        n = (n, n, n)
    nx, ny, nz = n
    rng = np.random.default_rng(seed)
    x = cell_centres(nx, 0, length)
    y = cell_centres(ny, 0, length)
    z = cell_centres(nz, 0, length)
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    prim = []
    for v in range(5):
        f = np.zeros_like(X)
        for _ in range(modes):
            kx, ky, kz = rng.integers(-2, 3, size=3)
            ph = rng.uniform(0, 2 * math.pi)
            f += rng.uniform(-1, 1) * np.cos(kx * X + ky * Y + kz * Z + ph)
        if v in (0, 4):
            prim.append(base[v] * (1.0 + amp * f))
        else:
            prim.append(base[v] + amp * f)
    dx = (length / nx, length / ny, length / nz)
    return np.ascontiguousarray(prim_to_cons(*prim, gamma=gamma)), dx


# ------------------------------------------------------------------------------------------------
# Channel flow (BASELINE config 4): [0, 2 pi H] x [-H, H] x [0, pi H], tanh-stretched y
# (b_g = 2), isothermal no-slip walls at y = -H, H, periodic x and z.  Units rho_b = U_b = H = 1.
# Bulk Re = 3000 (Re_tau ~ 180 by the H-series meshes) -> mu_w = 1/3000; bulk Mach 0.5
# (BASELINE config 4) -> T_w = (U_b/Ma)^2 / gamma in T = p/rho units; mu = mu_w (T/T_w)^0.7,
# Pr = 0.7.  Initial state: rho = 1, T = T_w, U = 1.5 (1 - y^2) plus 10% white noise
# of the local U, V and W white noise of 0.1 U_b, noise from a counter-based hash of
# (seed, global cell index) so the field does not depend on the decomposition.
# ------------------------------------------------------------------------------------------------
CHANNEL_SEED = 20220705


def channel_params(ma: float = 0.5, re_b: float = 3000.0, gamma: float = GAMMA):
    T_w = (1.0 / ma) ** 2 / gamma
    return dict(gamma=gamma, T_w=T_w, mu_w=1.0 / re_b, omega=0.7, prandtl=0.7, b_g=2.0,
                lo=(0.0, -1.0, 0.0), hi=(2 * math.pi, 1.0, math.pi), ma=ma, re_b=re_b)


def tanh_faces(n: int, lo: float, hi: float, b: float) -> np.ndarray:
    """Face coordinates of the tanh map: x_j = c + h tanh(b(2 j/n - 1))/tanh(b)."""
    s = np.arange(n + 1) / n
    return 0.5 * (lo + hi) + 0.5 * (hi - lo) * np.tanh(b * (2 * s - 1)) / np.tanh(b)


def _unit_noise(seed: int, idx: np.ndarray, stream: int) -> np.ndarray:
    """uniform [-1, 1) from splitmix64(seed, stream, global index): counter-based."""
    with np.errstate(over="ignore"):
        z = (idx.astype(np.uint64) + np.uint64(stream) * np.uint64(0x9E3779B97F4A7C15)
             + np.uint64(seed) * np.uint64(0xD1B54A32D192ED03))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) / float(1 << 53) * 2.0 - 1.0


def channel(n, z_begin: int = 0, nz_local: int | None = None, seed: int = CHANNEL_SEED, noise: float = 0.1,
            ma: float = 0.5, re_b: float = 3000.0, gamma: float = GAMMA):
    """Perturbed Poiseuille initial field of the channel (config 4).  Returns (q, params) with
    q [5][nz_local][ny][nx]; y cell centres are the midpoints of the tanh faces."""
    nx, ny, nz = n
    if nz_local is None:
        nz_local = nz - z_begin
    prm = channel_params(ma=ma, re_b=re_b, gamma=gamma)
    yf = tanh_faces(ny, -1.0, 1.0, prm["b_g"])
    yc = 0.5 * (yf[1:] + yf[:-1])
    k = np.arange(z_begin, z_begin + nz_local)
    K_, J_, I_ = np.meshgrid(k, np.arange(ny), np.arange(nx), indexing="ij")
    gid = (K_.astype(np.int64) * ny + J_) * nx + I_
    Y = yc[J_]
    Ub = 1.5 * (1.0 - Y * Y)
    U = Ub * (1.0 + noise * _unit_noise(seed, gid, 1))
    V = noise * _unit_noise(seed, gid, 2)
    W = noise * _unit_noise(seed, gid, 3)
    rho = np.ones_like(U)
    p = rho * prm["T_w"]
    return np.ascontiguousarray(prim_to_cons(rho, U, V, W, p, gamma)), prm
