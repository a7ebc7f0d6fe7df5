"""Pins of the oracle's x-z plane statistics (or_plane_stats, reading O-28).

Fields built from x and z harmonics over whole periods: on n >= 3 uniform points the discrete
means obey mean(cos) = mean(sin) = 0, mean(cos^2) = 1/2, and means of products of x- and
z-harmonics factor, so every moment has a closed form.  Profiles vary with y so an index slip
between planes shows."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_01173_b200 import inputs

GAMMA = 1.4
S = {k: i for i, k in enumerate(O.STAT_NAMES)}


def _field(nx=8, ny=5, nz=6, a=0.3, e=0.2, d=0.15):
    y = np.linspace(-0.8, 0.8, ny)
    r0 = 1.0 + 0.3 * y
    u0 = 1.5 * (1 - y ** 2)
    b = 0.1 + 0.2 * y
    p0 = 2.0 - 0.5 * y
    x = inputs.cell_centres(nx, 0, 2 * math.pi)
    z = inputs.cell_centres(nz, 0, math.pi) * 2  # one period of sin(z') over the plane
    Z, Y, X = np.meshgrid(z, np.arange(ny), x, indexing="ij")
    rho = r0[Y]
    U = u0[Y] + a * np.cos(X)
    V = b[Y] * np.cos(X) + d * np.sin(Z)
    W = e * np.cos(Z)
    q = inputs.prim_to_cons(rho, U, V, W, p0[Y], GAMMA)
    return q, dict(r0=r0, u0=u0, b=b, p0=p0, a=a, d=d, e=e)


def test_plane_means_closed_forms():
    q, f = _field()
    st = O.plane_stats(O.make_gas(), q, (1.0, 1.0, 1.0))
    r0, u0, b, p0, a, d, e = (f[k] for k in ("r0", "u0", "b", "p0", "a", "d", "e"))
    c0 = np.sqrt(GAMMA * p0 / r0)
    exact = {
        "rho": r0, "U": u0, "V": 0 * u0, "W": 0 * u0,
        "UU": u0 ** 2 + a * a / 2, "VV": b * b / 2 + d * d / 2, "WW": 0 * u0 + e * e / 2, "UV": a * b / 2,
        "rhoU": r0 * u0, "rhoV": 0 * u0, "rhoUV": r0 * a * b / 2,
        "c": c0, "MM": (u0 ** 2 + a * a / 2 + b * b / 2 + d * d / 2 + e * e / 2) / c0 ** 2, "T": p0 / r0, "p": p0,
    }
    for k, v in exact.items():
        np.testing.assert_allclose(st[:, S[k]], v, rtol=1e-13, atol=1e-15, err_msg=k)
    # Jensen: <M> <= sqrt(<M^2>), strict for a non-constant |U|
    assert np.all(st[:, S["M"]] < np.sqrt(st[:, S["MM"]]))


def test_mach_of_uniform_plane():
    q, f = _field(a=0.0, e=0.0, d=0.0)
    q[2] = 0.0  # V = 0 too (b cos x term)
    q[4] = f["p0"][None, :, None] / (GAMMA - 1) + 0.5 * q[1] ** 2 / q[0]
    st = O.plane_stats(O.make_gas(), q, (1.0, 1.0, 1.0))
    np.testing.assert_allclose(st[:, S["M"]], f["u0"] / np.sqrt(GAMMA * f["p0"] / f["r0"]), rtol=1e-14)
