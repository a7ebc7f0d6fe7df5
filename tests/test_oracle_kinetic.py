"""Pins of the oracle's kinetic machinery (A4-A6) against quadrature, closed forms and physics.

Nothing here re-types an oracle formula: moments and slopes are checked against brute-force
velocity-space quadrature (tests/kinetic_quadrature.py), the time integrals against scipy.quad,
the Gauss-point flux against (i) the Euler flux of a uniform state, (ii) the compressible
Navier-Stokes flux of the equilibrium limit, (iii) brute-force quadrature of
Eq. (6) with numerical time integration and a numpy 2x2 solve of Eq. (8)
(P:340-349), and (iv) mirror / tangential-swap symmetries.
"""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import oracle as O
from tests import kinetic_quadrature as KQ

K2 = O.K_of(1.4)


def test_internal_dof_gamma_1p4():
    # N = (5 - 3 gamma)/(gamma - 1) = 2 for gamma = 1.4 (O-20: fp64 gives 2 + 2 ulp)
    assert abs(K2 - 2.0) < 1e-14
    assert abs(O.K_of(5.0 / 3.0)) < 1e-14  # monatomic gas: no internal DOF


@pytest.mark.parametrize("which", [0, 1, -1])
def test_moments_vs_quadrature(which):
    rng = np.random.default_rng(11)
    for _ in range(12):
        U = rng.uniform(-3, 3)
        lam = math.exp(rng.uniform(math.log(0.1), math.log(10)))
        m = O.moments_u(U, lam, which)
        lo, hi = {0: (-np.inf, np.inf), 1: (0, np.inf), -1: (-np.inf, 0)}[which]
        for n in range(9):
            f = lambda u: u**n * math.sqrt(lam / math.pi) * math.exp(-lam * (u - U) ** 2)
            ref = integrate.quad(f, lo, hi, epsabs=0, epsrel=1e-13, limit=400)[0]
            # scale: the full-space absolute moment (half-space tails can be ~1e-16 of it)
            scale = integrate.quad(lambda u: abs(f(u)), -np.inf, np.inf, epsabs=0, epsrel=1e-13, limit=400)[0]
            assert abs(m[n] - ref) <= 1e-11 * scale, (which, n, U, lam)


def test_half_moment_additivity_and_symmetry():
    for U, lam in [(0.0, 1.0), (2.0, 1.0), (-0.7, 3.3)]:
        full, pos, neg = (O.moments_u(U, lam, w) for w in (0, 1, -1))
        np.testing.assert_allclose(pos + neg, full, rtol=1e-13, atol=1e-13)
    assert O.moments_u(0.0, 1.0, 1)[0] == pytest.approx(0.5, abs=1e-15)
    assert O.moments_u(0.0, 1.0, 0)[2] == pytest.approx(0.5, abs=1e-15)  # <u^2> = 1/(2 lam)


def test_psi_moments_vs_5d_quadrature():
    rng = np.random.default_rng(5)
    for which in (0, 1, -1):
        U, V, W = rng.normal(size=3)
        lam = rng.uniform(0.3, 3.0)
        mx = (1.0, U, V, W, lam)
        for (a, b, c, d) in [(0, 0, 0, 0), (1, 0, 0, 0), (2, 1, 0, 0), (1, 1, 1, 1), (2, 0, 2, 0), (3, 0, 1, 1)]:
            got = O.psi_moment(U, V, W, lam, K2, which, a, b, c, d)
            ref = KQ.moment(mx, lambda u, v, w, s: u**a * v**b * w**c * s**d * KQ.psi(u, v, w, s), which)
            np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-11 * np.abs(ref).max())


def test_maxwellian_reproduces_state():
    # moments of maxwellian_of(q) reproduce q
    q = np.array([1.3, 0.4, -0.2, 0.7, 3.1])
    mx = O.cons_to_maxw(q, K2)
    got = mx[0] * KQ.moment(mx, KQ.psi)
    np.testing.assert_allclose(got, q, rtol=1e-12)
    # (rho=1, m=0, rhoE=2.5) -> p = 1 -> lambda = rho/(2p) = 0.5 for gamma=1.4 (K=2; S:66 says 0.6: wrong, finding 9)
    assert O.cons_to_maxw([1, 0, 0, 0, 2.5], K2)[4] == pytest.approx(0.5, rel=1e-14)
    assert O.cons_to_maxw([1, 0, 0, 0, -1.0], K2) is None


def test_slope_solve_residual_by_quadrature():
    rng = np.random.default_rng(7)
    for _ in range(5):
        mx = np.array([1.0, *rng.normal(size=3), rng.uniform(0.2, 4.0)])
        b = rng.normal(size=5)
        a = O.slope_solve(mx, K2, b)
        res = KQ.moment(mx, lambda u, v, w, s: KQ.poly(a, u, v, w, s) * KQ.psi(u, v, w, s))
        np.testing.assert_allclose(res, b, rtol=1e-10, atol=1e-10 * np.abs(b).max())
    assert np.all(O.slope_solve(mx, K2, np.zeros(5)) == 0.0)


def _time_kernels(tau):
    e = lambda t: math.exp(-t / tau) if tau > 0 else 0.0
    return [
        lambda t: 1 - e(t),
        lambda t: (t + tau) * e(t) - tau,
        lambda t: t - tau + tau * e(t),
        lambda t: e(t),
        lambda t: -(tau + t) * e(t),
        lambda t: -tau * e(t),
    ]


@pytest.mark.parametrize("T,tau", [(1e-2, 3e-3), (7.1e-3, 8.75e-6), (0.5, 0.5), (1.0, 1e-3)])
def test_time_integrals_vs_quad(T, tau):
    g = O.time_integrals(T, tau)
    for k, f in enumerate(_time_kernels(tau)):
        ref = integrate.quad(f, 0, T, epsabs=0, epsrel=1e-13, limit=400, points=[min(T, 10 * tau)])[0]
        assert g[k] == pytest.approx(ref, rel=1e-10, abs=1e-16 * T), k


def test_time_integrals_euler_limit():
    # O-10: tau = 0 -> only the g0 and Abar g0 terms survive: gamma1 = T, gamma3 = T^2/2
    g = O.time_integrals(0.3, 0.0)
    np.testing.assert_array_equal(g, [0.3, 0.0, 0.5 * 0.3 * 0.3, 0.0, 0.0, 0.0])


def _prim_to_cons(rho, U, V, W, p, gamma=1.4):
    return np.array([rho, rho * U, rho * V, rho * W, p / (gamma - 1) + 0.5 * rho * (U * U + V * V + W * W)])


def test_euler_flux_of_uniform_state():
    # S:222 (tests/golden/spec_examples.txt): rho=1, U=(1,0,0), p=1 -> F = (1, 2, 0, 0, 4), dF = 0
    golden = [l.split() for l in open("tests/golden/spec_examples.txt") if l.startswith("euler_flux_uniform")][0]
    ref = np.array([float(x) for x in golden[1:6]])
    W = _prim_to_cons(1.0, 1.0, 0.0, 0.0, 1.0)
    z = np.zeros((3, 5))
    for mu in (0.0, 1e-3, 0.2):
        F, dF, tau = O.gp_flux(O.make_gas(mu=mu), W, z, W, z, z, 0.01)
        np.testing.assert_allclose(F, ref, rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(dF, 0.0, atol=1e-11)


def test_static_state_flux():
    # zero-velocity uniform state -> only the normal-momentum flux p survives
    W = _prim_to_cons(1.7, 0.0, 0.0, 0.0, 2.3)
    z = np.zeros((3, 5))
    F, dF, tau = O.gp_flux(O.make_gas(mu=1e-3), W, z, W, z, z, 0.02)
    np.testing.assert_allclose(F, [0, 2.3, 0, 0, 0], atol=1e-13)
    assert tau == pytest.approx(1e-3 / 2.3, rel=1e-14)  # tau = mu/p


def _ns_flux(prim, dprim, mu, K, gamma=1.4):
    """Compressible NS flux through an x-face: BGK transport coefficients
    mu = tau p, bulk-stress coefficient 2/(K+3), conductivity mu (K+5)/2 on T = p/rho."""
    rho, U, V, W, p = prim
    g = [dprim[i] for i in range(3)]  # g[i] = d(rho,U,V,W,p)/dx_i
    dU = np.array([[g[i][1 + j] for i in range(3)] for j in range(3)])  # dU[j][i] = dU_j/dx_i
    div = dU[0][0] + dU[1][1] + dU[2][2]
    sxx = mu * (2 * dU[0][0] - 2.0 / (K + 3) * div)
    sxy = mu * (dU[0][1] + dU[1][0])
    sxz = mu * (dU[0][2] + dU[2][0])
    dTdx = (g[0][4] * rho - p * g[0][0]) / rho**2
    qx = -mu * (K + 5) / 2 * dTdx
    E = p / (gamma - 1) + 0.5 * rho * (U * U + V * V + W * W)
    return np.array([rho * U, rho * U * U + p - sxx, rho * U * V - sxy, rho * U * W - sxz,
                     (E + p) * U - (U * sxx + V * sxy + W * sxz) + qx])


def _cons_grad(prim, dprim, gamma=1.4):
    rho, U, V, W, p = prim
    out = np.zeros((3, 5))
    for i in range(3):
        dr, dU, dV, dW, dp = dprim[i]
        out[i] = [dr, U * dr + rho * dU, V * dr + rho * dV, W * dr + rho * dW,
                  dp / (gamma - 1) + 0.5 * (U * U + V * V + W * W) * dr + rho * (U * dU + V * dV + W * dW)]
    return out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_navier_stokes_limit(seed):
    # O-P5: g_l = g_r = g0 with equal slopes -> f = g0 [1 - tau(a.u + A) + t A] (Eq. 6 collapses),
    # whose flux is the NS flux with the BGK transport coefficients.
    rng = np.random.default_rng(seed)
    prim = np.array([rng.uniform(0.5, 2), *rng.normal(scale=0.5, size=3), rng.uniform(0.5, 3)])
    dprim = rng.normal(scale=0.3, size=(3, 5))
    W = _prim_to_cons(*prim)
    dW = _cons_grad(prim, dprim)
    mu = 10 ** rng.uniform(-4, -2)
    dt = 10 ** rng.uniform(-3, -1)
    F, dF, tau = O.gp_flux(O.make_gas(mu=mu), W, dW, W, dW, dW, dt)
    ref = _ns_flux(prim, dprim, tau * prim[4], K2)
    np.testing.assert_allclose(F, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())


def _brute_force_flux(Wl, dWl, Wr, dWr, dW0, dt, mu):
    """Eq. (6) integrated over velocity space by quadrature and over [0,T] by scipy.quad,
    then Eq. (8) solved with numpy: completely independent of the oracle's algebra."""
    ml, mr = KQ.maxwellian_of(Wl), KQ.maxwellian_of(Wr)
    Q0 = ml[0] * KQ.moment(ml, KQ.psi, +1) + mr[0] * KQ.moment(mr, KQ.psi, -1)
    m0 = KQ.maxwellian_of(Q0)
    np.testing.assert_allclose(m0[0] * KQ.moment(m0, KQ.psi), Q0, rtol=1e-12)
    tau = mu / (m0[0] / (2 * m0[4]))
    al, Al = KQ.slopes(ml, dWl)
    ar, Ar = KQ.slopes(mr, dWr)
    ab, Ab = KQ.slopes(m0, dW0)

    def au(a, u, v, w, s):  # a1.psi u + a2.psi v + a3.psi w
        return KQ.poly(a[0], u, v, w, s) * u + KQ.poly(a[1], u, v, w, s) * v + KQ.poly(a[2], u, v, w, s) * w

    P = lambda f: (lambda u, v, w, s: u * f(u, v, w, s) * KQ.psi(u, v, w, s))
    one = lambda u, v, w, s: np.ones_like(u)
    Phi = [
        m0[0] * KQ.moment(m0, P(one)),
        m0[0] * KQ.moment(m0, P(lambda u, v, w, s: au(ab, u, v, w, s))),
        m0[0] * KQ.moment(m0, P(lambda u, v, w, s: KQ.poly(Ab, u, v, w, s))),
        ml[0] * KQ.moment(ml, P(one), +1) + mr[0] * KQ.moment(mr, P(one), -1),
        ml[0] * KQ.moment(ml, P(lambda u, v, w, s: au(al, u, v, w, s)), +1)
        + mr[0] * KQ.moment(mr, P(lambda u, v, w, s: au(ar, u, v, w, s)), -1),
        ml[0] * KQ.moment(ml, P(lambda u, v, w, s: KQ.poly(Al, u, v, w, s)), +1)
        + mr[0] * KQ.moment(mr, P(lambda u, v, w, s: KQ.poly(Ar, u, v, w, s)), -1),
    ]
    kern = _time_kernels(tau)

    def I(T):
        return sum(integrate.quad(kern[k], 0, T, epsabs=0, epsrel=1e-13, limit=400)[0] * Phi[k] for k in range(6))

    Ifull, Ihalf = I(dt), I(dt / 2)
    A = np.array([[dt, 0.5 * dt * dt], [0.5 * dt, dt * dt / 8]])
    sol = np.linalg.solve(A, np.stack([Ifull, Ihalf]))
    return sol[0], sol[1], tau


@pytest.mark.parametrize("seed,tau_ratio", [(0, 0.3), (1, 0.05), (2, 2.0)])
def test_gp_flux_vs_bruteforce_quadrature(seed, tau_ratio):
    rng = np.random.default_rng(100 + seed)
    pl = np.array([rng.uniform(0.8, 1.5), *rng.normal(scale=0.4, size=3), rng.uniform(0.6, 2.0)])
    pr = pl * (1 + rng.normal(scale=0.1, size=5))
    pr[1:4] = pl[1:4] + rng.normal(scale=0.2, size=3)
    Wl, Wr = _prim_to_cons(*pl), _prim_to_cons(*pr)
    dWl, dWr, dW0 = (rng.normal(scale=0.2, size=(3, 5)) * np.abs(Wl) for _ in range(3))
    dt = 0.02
    p0_guess = 0.5 * (pl[4] + pr[4])
    mu = tau_ratio * dt * p0_guess
    F, dF, tau = O.gp_flux(O.make_gas(mu=mu), Wl, dWl, Wr, dWr, dW0, dt)
    Fr, dFr, taur = _brute_force_flux(Wl, dWl, Wr, dWr, dW0, dt, mu)
    assert tau == pytest.approx(taur, rel=1e-11)
    np.testing.assert_allclose(F, Fr, rtol=1e-9, atol=1e-9 * np.abs(Fr).max())
    np.testing.assert_allclose(dF, dFr, rtol=1e-8, atol=1e-8 * np.abs(dFr).max())


def _mirror(v):
    return v * np.array([1, -1, 1, 1, 1])


def test_flux_mirror_and_tangential_swap_symmetry():
    rng = np.random.default_rng(3)
    pl = np.array([1.1, 0.3, -0.2, 0.4, 1.3])
    pr = np.array([0.9, -0.1, 0.25, 0.1, 1.1])
    Wl, Wr = _prim_to_cons(*pl), _prim_to_cons(*pr)
    dWl, dWr, dW0 = (rng.normal(scale=0.2, size=(3, 5)) for _ in range(3))
    gas = O.make_gas(mu=2e-3)
    F, dF, _ = O.gp_flux(gas, Wl, dWl, Wr, dWr, dW0, 0.01)
    # x -> -x: left/right swap, normal momentum and normal derivatives flip
    md = lambda d: np.stack([-_mirror(d[0]), _mirror(d[1]), _mirror(d[2])])
    Fm, dFm, _ = O.gp_flux(gas, _mirror(Wr), md(dWr), _mirror(Wl), md(dWl), md(dW0), 0.01)
    sgn = np.array([-1, 1, -1, -1, -1])
    np.testing.assert_allclose(Fm, sgn * F, rtol=1e-12, atol=1e-13 * np.abs(F).max())
    np.testing.assert_allclose(dFm, sgn * dF, rtol=1e-10, atol=1e-11 * np.abs(dF).max())
    # t1 <-> t2: swap v,w components and the two tangential derivative directions
    sw = lambda v: v[[0, 1, 3, 2, 4]]
    sd = lambda d: np.stack([sw(d[0]), sw(d[2]), sw(d[1])])
    Fs, dFs, _ = O.gp_flux(gas, sw(Wl), sd(dWl), sw(Wr), sd(dWr), sd(dW0), 0.01)
    np.testing.assert_allclose(Fs, sw(F), rtol=1e-13, atol=1e-14 * np.abs(F).max())
    np.testing.assert_allclose(dFs, sw(dF), rtol=1e-12, atol=1e-13 * np.abs(dF).max())


def test_tgv_collision_time():
    # TGV mu = 1/1600, p0 = 100/1.4 -> tau0 = 8.75e-6
    p0 = 100 / 1.4
    W = _prim_to_cons(1.0, 0.0, 0.0, 0.0, p0)
    z = np.zeros((3, 5))
    _, _, tau = O.gp_flux(O.make_gas(mu=1 / 1600), W, z, W, z, z, 1e-3)
    assert tau == pytest.approx(8.75e-6, rel=1e-13)
