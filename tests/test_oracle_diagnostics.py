"""Pins of the oracle's volume diagnostics (or_diagnostics, readings O-24, O-25)
against closed forms that do not use the oracle:

* TGV velocity field with rho = 1 on [-pi, pi]^3: on n uniform points per period the cell mean of
  a product of squared first harmonics is exactly 1/8, and the fourth-order central difference
  maps sin/cos of unit wavenumber onto cos/-sin times kappa(h) = (8 sin h - sin 2h) / (6 h)
  exactly, so E_k, zeta, eps_s and eps_d have closed forms in kappa_x, kappa_y, kappa_z.
  Different n per axis makes every axis-index slip visible.
* a linear shear U = a y on a tanh-stretched y axis (metric J at the cell centre, O-18/O-25).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_01173_b200 import inputs

E, Z, ES, ED, MASS, MX, MY, MZ, EN, VOL, PDIL = range(11)


def kappa(h):
    return (8 * math.sin(h) - math.sin(2 * h)) / (6 * h)


def _tgv_rho1(n, rho=1.0):
    nx, ny, nz = n
    x = inputs.cell_centres(nx, -math.pi, math.pi)
    y = inputs.cell_centres(ny, -math.pi, math.pi)
    z = inputs.cell_centres(nz, -math.pi, math.pi)
    Zg, Yg, Xg = np.meshgrid(z, y, x, indexing="ij")
    U = np.sin(Xg) * np.cos(Yg) * np.cos(Zg)
    V = -np.cos(Xg) * np.sin(Yg) * np.cos(Zg)
    return inputs.prim_to_cons(np.full(U.shape, rho), U, V, 0 * U, 1.0 + 0 * U)


@pytest.mark.parametrize("n", [(16, 16, 16), (12, 16, 20)])
def test_tgv_closed_forms(n):
    q = _tgv_rho1(n)
    mu = 0.01
    h = [2 * math.pi / m for m in n]
    kx, ky, kz = (kappa(v) for v in h)
    d = O.diagnostics(O.make_gas(mu=mu), q, tuple(h))
    assert d[E] == pytest.approx(1 / 8, rel=1e-14)
    om2 = (2 * kz * kz + (kx + ky) ** 2) / 8           # mean |omega|^2
    assert d[Z] == pytest.approx(0.5 * om2, rel=1e-13)
    assert d[ES] == pytest.approx(mu * om2, rel=1e-13)
    assert d[ED] == pytest.approx(4 / 3 * mu * (kx - ky) ** 2 / 8, rel=1e-12, abs=1e-20)
    # sums of n^3 equal terms: rounding grows like n^3 eps
    assert d[VOL] == pytest.approx((2 * math.pi) ** 3, rel=1e-12)
    assert d[MASS] == pytest.approx((2 * math.pi) ** 3, rel=1e-12)
    assert abs(d[MX]) < 1e-12 and abs(d[MY]) < 1e-12 and d[MZ] == 0.0


def test_tgv_density_scaling():
    """rho = 2 everywhere with rho0 = 2: E_k and zeta unchanged; eps_s, eps_d halve (1/rho0)."""
    n = (12, 12, 12)
    h = (2 * math.pi / 12,) * 3
    d1 = O.diagnostics(O.make_gas(mu=0.1), _tgv_rho1(n), h)
    d2 = O.diagnostics(O.make_gas(mu=0.1), _tgv_rho1(n, rho=2.0), h, rho0=2.0)
    assert d2[E] == pytest.approx(d1[E], rel=1e-14)
    assert d2[Z] == pytest.approx(d1[Z], rel=1e-14)
    assert d2[ES] == pytest.approx(0.5 * d1[ES], rel=1e-14)
    assert d2[MASS] == pytest.approx(2 * d1[MASS], rel=1e-14)


def test_potential_flow():
    """U = sin x: omega = 0 exactly, (div U)^2 mean = kappa^2 / 2."""
    n = 10
    h = 2 * math.pi / n
    x = inputs.cell_centres(n, -math.pi, math.pi)
    U = np.broadcast_to(np.sin(x), (n, n, n))
    q = inputs.prim_to_cons(np.ones((n, n, n)), U, 0 * U, 0 * U, 1.0 + 0 * U)
    d = O.diagnostics(O.make_gas(mu=0.3), q, (h, h, h))
    assert d[ES] == 0.0 and d[Z] == 0.0
    assert d[ED] == pytest.approx(4 / 3 * 0.3 * kappa(h) ** 2 / 2, rel=1e-13)
    assert abs(d[PDIL]) < 1e-14  # uniform p: mean of div U = kappa mean(cos x) = 0


@pytest.mark.parametrize("n", [8, 10, 13])
def test_pressure_dilatation_closed_form(n):
    """U = sin x, p = 1 + 0.5 cos x, rho = 1.3: the discrete div U is kappa(h) cos x exactly, so
    sum p div U dV / Omega = kappa (mean cos x + 0.5 mean cos^2 x) = kappa/4 (discrete orthogonality,
    n >= 3), and Pi = kappa/(4 rho0).  A dropped (gamma - 1), a kinetic-energy slip in p or a wrong
    sign all fail."""
    h = 2 * math.pi / n
    x = inputs.cell_centres(n, -math.pi, math.pi)
    U = np.broadcast_to(np.sin(x), (n, n, n))
    p = np.broadcast_to(1.0 + 0.5 * np.cos(x), (n, n, n))
    q = inputs.prim_to_cons(np.full((n, n, n), 1.3), U, 0 * U, 0 * U, p)
    d = O.diagnostics(O.make_gas(mu=0.0), q, (h, h, h), rho0=1.3)
    assert d[PDIL] == pytest.approx(kappa(h) / 4 / 1.3, rel=1e-12)
    d2 = O.diagnostics(O.make_gas(mu=0.0), q, (h, h, h), rho0=1.0)
    assert d2[PDIL] == pytest.approx(kappa(h) / 4, rel=1e-12)


def test_linear_shear_on_tanh_axis():
    """U = a y on the channel's tanh-stretched y axis (ghosts supplied from the analytic map): the
    derivative is a to the difference's O(h^4) error; J taken at a face instead of the centre
    would be off by O(h)."""
    nx, ny, nz = 6, 64, 6
    ch = inputs.channel_params()
    b = ch["b_g"]
    gr = O.make_grid((nx, ny, nz), (2 * math.pi / nx, 0.0, math.pi / nz), bc=(0, 2, 0), stretch=(0, 1, 0),
                     lo=ch["lo"], hi=ch["hi"], stretch_b=(0, b, 0))
    jj = np.arange(-3, ny + 3) + 0.5
    yc = np.tanh(b * (2 * jj / ny - 1)) / math.tanh(b)   # analytic map at cell-centre indices
    a = 0.7
    qg = np.zeros((5, nz + 6, ny + 6, nx + 6))
    qg[0] = 1.0
    qg[1] = a * yc[None, :, None]
    qg[4] = 2.5 + 0.5 * qg[1] ** 2
    O.lib().or_fill_ghosts(O.C.byref(O.make_gas()), O.C.byref(gr), O._p(qg))
    mu = 0.05
    d = O.diagnostics(O.make_gas(mu=mu), qg=qg, grid=gr)
    assert d[VOL] == pytest.approx(2 * math.pi * 2.0 * math.pi, rel=1e-12)
    assert d[ES] == pytest.approx(mu * a * a, rel=5e-6)  # measured 4.6e-7; face-J would be ~6e-2
    assert d[ED] == 0.0


def test_matches_harness_on_uniform_grid():
    """tests/diagnostics.py (numpy, periodic rolls) and the oracle give the same E_k and zeta on
    the TGV initial field (same definitions, independent code)."""
    from tests import diagnostics as D
    q, dx = inputs.tgv(16)
    d = O.diagnostics(O.make_gas(mu=1 / 1600), q, dx)
    assert d[E] == pytest.approx(D.kinetic_energy(q), rel=1e-13)
    assert d[Z] == pytest.approx(D.enstrophy(q, dx), rel=1e-12)
