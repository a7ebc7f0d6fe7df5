"""Pins of the oracle's reconstruction (A2-A3; readings O-1, O-3, O-4, O-6, O-8).

Checked against: exact polynomial data (analytic cell averages), sympy-exact quartic weights
(A.9, computed here symbolically, not by the oracle's linear solve), WENO constant/linear
exactness and observed order, and the WENO-Z linear-weight limit.
"""
import math

import numpy as np
import pytest
import sympy as sp

from oracle import oracle as O


def test_weno_constant_and_linear_exact():
    # exact up to rounding of the candidate coefficients (they do not sum to 1 bitwise in fp64);
    # bitwise preservation of uniform flow is a whole-step property (O-P1, test_oracle_step.py)
    for c in (0.0, 1.0, -3.7, 178.6):
        assert O.weno5z([c] * 5, "right") == pytest.approx(c, rel=4e-16, abs=0)
        assert O.weno5z([c] * 5, "left") == pytest.approx(c, rel=4e-16, abs=0)
    # cell averages of f(x) = 2 + 3x on cells [m-1/2, m+1/2] are f(m): right edge = f(1/2)
    q = [2 + 3 * m for m in range(-2, 3)]
    assert O.weno5z(q, "right") == pytest.approx(3.5, abs=1e-14)
    assert O.weno5z(q, "left") == pytest.approx(0.5, abs=1e-14)


def test_weno_smooth_limit_is_linear_fifth_order_value():
    # For smooth data the WENO-Z weights tend to (0.1, 0.6, 0.3) and the edge value to the
    # 5-cell quartic edge value (1/30, -13/60, 47/60, 9/20, -1/20) (A.9; sympy below).
    x = sp.symbols("x")
    c = sp.symbols("c0:5")
    P = sum(c[i] * x**i for i in range(5))
    qs = sp.symbols("q0:5")
    sol = sp.solve([sp.integrate(P, (x, m - sp.Rational(1, 2), m + sp.Rational(1, 2))) - qs[m + 2]
                    for m in range(-2, 3)], c)
    edge = sp.expand(P.subs(sol).subs(x, sp.Rational(1, 2)))
    w = np.array([float(edge.coeff(q)) for q in qs])
    np.testing.assert_allclose(w, [1 / 30, -13 / 60, 47 / 60, 9 / 20, -1 / 20], rtol=1e-15)
    h = 1e-2
    q = np.array([(math.cos((m - 0.5) * h) - math.cos((m + 0.5) * h)) / h for m in range(-2, 3)])
    # WENO-Z deviates from the linear value by O(h^6) * scale here
    assert abs(O.weno5z(q, "right") - w @ q) < 1e-12


def test_weno_order_on_sine():
    errs = []
    for n in (16, 32, 64, 128):
        h = 2 * math.pi / n
        avg = lambda m: (math.cos(m * h) - math.cos((m + 1) * h)) / h  # average of sin on [mh,(m+1)h]
        e = 0.0
        for i in range(n):
            q = [avg(i + s) for s in range(-2, 3)]
            e = max(e, abs(O.weno5z(q, "right") - math.sin((i + 1) * h)))
            e = max(e, abs(O.weno5z(q, "left") - math.sin(i * h)))
        errs.append(e)
    orders = [math.log2(errs[k] / errs[k + 1]) for k in range(3)]
    assert min(orders[1:]) >= 4.5, orders


def _poly_avg(coef, lo, hi):
    """exact average of sum coef[p] x^p over [lo, hi]"""
    return sum(c * (hi ** (p + 1) - lo ** (p + 1)) / (p + 1) for p, c in enumerate(coef)) / (hi - lo)


def _poly_val(coef, x, der=False):
    if der:
        return sum(p * c * x ** (p - 1) for p, c in enumerate(coef) if p > 0)
    return sum(c * x**p for p, c in enumerate(coef))


def test_face_gauss_points_exact_on_separable_polynomials():
    """f = g(n) a(t1) b(t2) with g linear (WENO and the O-3 slope are exact on it) and a, b
    quartic (the O-4 tangential operator is exact to degree 4): every Gauss-point input must
    equal the analytic value.  Also pins the Gauss abscissae -+sqrt(3)/6 (O-8) and the
    O-6 equilibrium derivatives."""
    h = np.array([0.3, 0.2, 0.25])
    rng = np.random.default_rng(2)
    g = [1.3, 0.7]
    A = rng.normal(size=5)
    B = rng.normal(size=5)
    comp_scale = np.array([1.0, 0.3, -0.5, 2.0, 4.0])
    cells = np.zeros((6, 5, 5, 5))
    for n in range(6):
        # cell n covers [(n-3) h_n, (n-2) h_n]; the face is at 0
        gn = _poly_avg(g, (n - 3) * h[0], (n - 2) * h[0])
        for a in range(5):
            ta = _poly_avg(A, (a - 2.5) * h[1], (a - 1.5) * h[1])
            for b in range(5):
                tb = _poly_avg(B, (b - 2.5) * h[2], (b - 1.5) * h[2])
                cells[n, a, b, :] = comp_scale * gn * ta * tb
    out = O.face_gauss_points(cells, h)
    s = math.sqrt(3) / 6
    for m in range(2):
        for nn in range(2):
            gp = 2 * m + nn
            y = (-s if m == 0 else s) * h[1]
            z = (-s if nn == 0 else s) * h[2]
            val = _poly_val(g, 0.0) * _poly_val(A, y) * _poly_val(B, z)
            dn = _poly_val(g, 0.0, True) * _poly_val(A, y) * _poly_val(B, z)
            d1 = _poly_val(g, 0.0) * _poly_val(A, y, True) * _poly_val(B, z)
            d2 = _poly_val(g, 0.0) * _poly_val(A, y) * _poly_val(B, z, True)
            exp_val = comp_scale * val
            tol = 1e-11 * np.abs(comp_scale).max() * (1 + abs(val) + abs(dn) + abs(d1) + abs(d2))
            for key in ("Wl", "Wr"):
                np.testing.assert_allclose(out[key][gp], exp_val, atol=tol)
            for key in ("dWl", "dWr", "dW0"):
                np.testing.assert_allclose(out[key][gp][0], comp_scale * dn, atol=tol)
                np.testing.assert_allclose(out[key][gp][1], comp_scale * d1, atol=tol)
                np.testing.assert_allclose(out[key][gp][2], comp_scale * d2, atol=tol)


def test_face_gauss_points_constant_field():
    cells = np.ones((6, 5, 5, 5)) * np.array([1.0, 0.2, 0.3, -0.1, 2.5])
    out = O.face_gauss_points(cells, [0.1, 0.1, 0.1])
    for gp in range(4):
        np.testing.assert_allclose(out["Wl"][gp], cells[0, 0, 0], rtol=2e-15)
        np.testing.assert_allclose(out["Wr"][gp], cells[0, 0, 0], rtol=2e-15)
    for key in ("dWl", "dWr", "dW0"):
        assert np.abs(out[key]).max() < 1e-12


def test_normal_slope_reading_O3_and_O6():
    """O-3: slope of the left state = derivative at x=1/2 of the parabola with edge values A, B
    and mean M; O-6: D is the edge derivative of the 5-cell quartic (A.9) -> exact on a cubic's
    cell averages across the face.  Cubic data along the normal, constant tangentially."""
    h = np.array([0.5, 1.0, 1.0])
    cub = [0.3, -1.2, 0.8, 0.5]
    cells = np.zeros((6, 5, 5, 5))
    for n in range(6):
        cells[n] = _poly_avg(cub, (n - 3) * h[0], (n - 2) * h[0])
    out = O.face_gauss_points(cells, h)
    # D (4-point central derivative) is exact for cubics: d/dx at the face x=0
    np.testing.assert_allclose(out["dW0"][0][0], _poly_val(cub, 0.0, True), rtol=1e-12)
