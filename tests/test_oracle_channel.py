"""Pins of the oracle's channel-flow machinery (readings O-12, O-17, O-18):
the tanh mesh against the paper's Tables 6-7, the analytic metric against finite differences of the
face map, the power-law / Pr = 0.7 Gauss-point flux against the Navier-Stokes limit and a
brute-force quadrature of Eq. (6) with the heat-flux correction, and the isothermal-wall ghosts
against rest-state preservation, the wall mass flux and the y-reflection symmetry."""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import oracle as O
from paper_2207_01173_b200 import inputs
from tests import kinetic_quadrature as KQ
from tests.test_oracle_kinetic import _cons_grad, _ns_flux, _prim_to_cons, _time_kernels

K2 = O.K_of(1.4)
CH = inputs.channel_params()


def _channel_grid(n, lo=(0.0, -1.0, 0.0), hi=(2 * math.pi, 1.0, math.pi), b=2.0):
    dx = ((hi[0] - lo[0]) / n[0], 0.0, (hi[2] - lo[2]) / n[2])
    return O.make_grid(n, dx, bc=(0, 1, 0), stretch=(0, 1, 0), lo=lo, hi=hi, stretch_b=(0, b, 0))


def test_channel_mesh_tables_6_7():
    rows = [l.split() for l in open("tests/golden/tables67_channel_mesh.txt") if l.strip() and not l.startswith("#")]
    for case, nx, ny, nz, ymin, ymax, dxp, dzp in rows:
        nx, ny, nz = int(nx), int(ny), int(nz)
        gr = _channel_grid((nx, ny, nz))
        yf = O.axis_faces(gr, 1)
        assert yf[0] == pytest.approx(-1.0, abs=1e-15) and yf[-1] == pytest.approx(1.0, abs=1e-15)
        dy = np.diff(yf)
        if case.startswith("G"):
            # the table's digits are truncated, not rounded (G2: 0.4592 -> 0.45; the others agree
            # either way): compare floor(100 x)/100
            re_tau = 395.0
            trunc = lambda x: math.floor(x * 100 + 1e-9) / 100
            assert trunc(dy.min() * re_tau) == float(ymin), case
            assert trunc(dy.max() * re_tau) == float(ymax), case
            assert trunc(2 * math.pi / nx * re_tau) == float(dxp)
            assert trunc(math.pi / nz * re_tau) == float(dzp)
        else:  # H: Re_tau implied by Delta x+; the paper's wall units differ by a few % (SURVEY O-P14)
            re_tau = float(dxp) * nx / (2 * math.pi)
            assert math.pi / nz * re_tau == pytest.approx(float(dzp), rel=2e-3)
            assert dy.min() * re_tau == pytest.approx(float(ymin), rel=0.06)
            assert dy.max() * re_tau == pytest.approx(float(ymax), rel=0.06)


def test_metric_matches_finite_differences_of_the_map():
    gr = _channel_grid((8, 64, 8))
    yf = O.axis_faces(gr, 1)
    for j in (0, 5, 31, 32, 63):
        # J = d zeta / dy: compare with 1 / (dy/dzeta) from face differences (O(h^2))
        dyz = yf[j + 1] - yf[j]
        assert O.axis_metric(gr, 1, j + 0.5) == pytest.approx(1.0 / dyz, rel=2e-3)
    # uniform axes: J = 1/dx exactly
    assert O.axis_metric(gr, 0, 3.3) == pytest.approx(8 / (2 * math.pi), rel=1e-15)


@pytest.mark.parametrize("seed", [0, 1])
def test_navier_stokes_limit_power_law_prandtl(seed):
    # O-P5 with the config-4 transport: tau = mu(T0)/p0, mu = mu_w (T/T_w)^0.7, and the O-12 fix
    # turning the BGK conductivity mu (K+5)/2 into mu (K+5)/(2 Pr)
    rng = np.random.default_rng(seed)
    prim = np.array([rng.uniform(0.7, 1.4), *rng.normal(scale=0.5, size=3), rng.uniform(2.0, 3.5)])
    dprim = rng.normal(scale=0.3, size=(3, 5))
    W = _prim_to_cons(*prim)
    dW = _cons_grad(prim, dprim)
    gas = O.make_gas(mu=1 / 3000, mu_law=1, T_ref=CH["T_w"], omega=0.7, prandtl=0.7)
    F, dF, tau = O.gp_flux(gas, W, dW, W, dW, dW, 0.01)
    T = prim[4] / prim[0]
    mu = (1 / 3000) * (T / CH["T_w"]) ** 0.7
    assert tau == pytest.approx(mu / prim[4], rel=1e-12)
    ref = _ns_flux(prim, dprim, mu, K2)
    # the Pr fix scales the Fourier term by 1/Pr
    rho, U, V, Wv, p = prim
    dTdx = (dprim[0][4] * rho - p * dprim[0][0]) / rho**2
    ref[4] += -(mu * (K2 + 5) / 2) * dTdx * (1 / 0.7 - 1)
    np.testing.assert_allclose(F, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())


def _heat_flux_quadrature(Wl, dWl, Wr, dWr, dW0, dt, mu):
    """q(t) = int (u-U0) (|u-U0|^2 + xi^2)/2 f dXi of Eq. (6), integrated over both windows by
    brute-force quadrature, then linearised by Eq. (8)."""
    ml, mr = KQ.maxwellian_of(Wl), KQ.maxwellian_of(Wr)
    Q0 = ml[0] * KQ.moment(ml, KQ.psi, +1) + mr[0] * KQ.moment(mr, KQ.psi, -1)
    m0 = KQ.maxwellian_of(Q0)
    U0 = m0[1:4]
    tau = mu / (m0[0] / (2 * m0[4]))
    al, Al = KQ.slopes(ml, dWl)
    ar, Ar = KQ.slopes(mr, dWr)
    ab, Ab = KQ.slopes(m0, dW0)

    def au(a, u, v, w, s):
        return KQ.poly(a[0], u, v, w, s) * u + KQ.poly(a[1], u, v, w, s) * v + KQ.poly(a[2], u, v, w, s) * w

    def hq(f):
        return lambda u, v, w, s: f(u, v, w, s) * (u - U0[0]) * 0.5 * ((u - U0[0]) ** 2 + (v - U0[1]) ** 2 + (w - U0[2]) ** 2 + s)

    one = lambda u, v, w, s: np.ones_like(u)
    Phi = [
        m0[0] * KQ.moment(m0, hq(one)),
        m0[0] * KQ.moment(m0, hq(lambda u, v, w, s: au(ab, u, v, w, s))),
        m0[0] * KQ.moment(m0, hq(lambda u, v, w, s: KQ.poly(Ab, u, v, w, s))),
        ml[0] * KQ.moment(ml, hq(one), +1) + mr[0] * KQ.moment(mr, hq(one), -1),
        ml[0] * KQ.moment(ml, hq(lambda u, v, w, s: au(al, u, v, w, s)), +1)
        + mr[0] * KQ.moment(mr, hq(lambda u, v, w, s: au(ar, u, v, w, s)), -1),
        ml[0] * KQ.moment(ml, hq(lambda u, v, w, s: KQ.poly(Al, u, v, w, s)), +1)
        + mr[0] * KQ.moment(mr, hq(lambda u, v, w, s: KQ.poly(Ar, u, v, w, s)), -1),
    ]
    kern = _time_kernels(tau)
    I = lambda T: sum(integrate.quad(kern[k], 0, T, epsabs=0, epsrel=1e-13, limit=400)[0] * Phi[k] for k in range(6))
    A = np.array([[dt, 0.5 * dt * dt], [0.5 * dt, dt * dt / 8]])
    return np.linalg.solve(A, np.array([I(dt), I(dt / 2)]))


@pytest.mark.parametrize("seed", [0, 1])
def test_prandtl_fix_vs_bruteforce_quadrature(seed):
    rng = np.random.default_rng(300 + seed)
    pl = np.array([rng.uniform(0.8, 1.5), *rng.normal(scale=0.4, size=3), rng.uniform(0.6, 2.0)])
    pr = pl * (1 + rng.normal(scale=0.1, size=5))
    pr[1:4] = pl[1:4] + rng.normal(scale=0.2, size=3)
    Wl, Wr = _prim_to_cons(*pl), _prim_to_cons(*pr)
    dWl, dWr, dW0 = (rng.normal(scale=0.2, size=(3, 5)) * np.abs(Wl) for _ in range(3))
    dt, mu, Pr = 0.02, 0.2 * 0.02 * pl[4], 0.7
    F1, dF1, _ = O.gp_flux(O.make_gas(mu=mu), Wl, dWl, Wr, dWr, dW0, dt)
    Fp, dFp, _ = O.gp_flux(O.make_gas(mu=mu, prandtl=Pr), Wl, dWl, Wr, dWr, dW0, dt)
    qn, dqn = _heat_flux_quadrature(Wl, dWl, Wr, dWr, dW0, dt, mu)
    np.testing.assert_allclose(Fp[:4], F1[:4], rtol=0, atol=0)
    assert Fp[4] == pytest.approx(F1[4] + (1 / Pr - 1) * qn, rel=1e-9, abs=1e-9 * abs(F1[4]))
    assert dFp[4] == pytest.approx(dF1[4] + (1 / Pr - 1) * dqn, rel=1e-8, abs=1e-8 * abs(dF1[4]))


def _rest_state(n, T_w, rho=1.3):
    return inputs.uniform(n, rho=rho, vel=(0.0, 0.0, 0.0), p=rho * T_w)


def test_gas_at_rest_between_isothermal_walls_is_steady():
    n = (6, 12, 5)
    gr = _channel_grid(n)
    gas = O.make_gas(mu=1 / 3000, mu_law=1, T_ref=CH["T_w"], omega=0.7, prandtl=0.7, T_wall=CH["T_w"])
    q = _rest_state(n, CH["T_w"])
    q2, _ = O.run(gas, q, None, 2, dt_fixed=1e-3, grid=gr)
    np.testing.assert_array_equal(q2, q)


def test_wall_ghosts_mirror_and_zero_wall_mass_flux():
    n = (6, 16, 5)
    gr = _channel_grid(n)
    gas = O.make_gas(mu=1 / 3000, mu_law=1, T_ref=CH["T_w"], omega=0.7, prandtl=0.7, T_wall=CH["T_w"])
    q, _ = inputs.channel(n)  # isothermal (T = T_w) perturbed Poiseuille field
    qg = O.ghosted(q, gas=gas, grid=gr)
    # O-17 mirror: rho and rhoE reflect, momenta flip sign, across both walls (T = T_w here)
    g = 3
    for m in range(3):
        for side_g, side_i in ((g - 1 - m, g + m), (g + n[1] + m, g + n[1] - 1 - m)):
            np.testing.assert_allclose(qg[[0, 4], g:-g, side_g, g:-g], qg[[0, 4], g:-g, side_i, g:-g], rtol=1e-14)
            np.testing.assert_allclose(qg[1:4, g:-g, side_g, g:-g], -qg[1:4, g:-g, side_i, g:-g], rtol=1e-14)
    # no mass through the walls.  Exact only when the near-wall tangential velocity vanishes: the
    # no-slip mirror also flips U and W, so (Q^l, Q^r) at the wall is a geometric mirror pair only
    # for purely wall-normal motion.  With V-only perturbations the total mass is conserved to
    # round-off; with the full field the wall mass flux is a small discretisation error.
    rho = q[0]
    qv = inputs.prim_to_cons(rho, 0 * rho, q[2] / rho, 0 * rho, rho * CH["T_w"])
    vol = np.diff(O.axis_faces(gr, 1))[None, :, None] * gr.dx[0] * gr.dx[2]
    Lv, _ = O.operator(gas, np.ascontiguousarray(qv), None, 1e-3, grid=gr)
    assert abs(math.fsum((Lv[0] * vol).ravel())) <= 1e-13 * math.fsum((np.abs(Lv[0]) * vol).ravel())
    L, dL = O.operator(gas, q, None, 1e-3, grid=gr)
    total, scale = math.fsum((L[0] * vol).ravel()), math.fsum((np.abs(L[0]) * vol).ravel())
    assert abs(total) <= 1e-6 * scale
    # momentum is not conserved (wall shear): the x-momentum total is O(1) of its scale
    assert abs(math.fsum((L[1] * vol).ravel())) > 1e-3 * math.fsum((np.abs(L[1]) * vol).ravel())


def test_channel_reflection_symmetry():
    # y -> -y maps the stretched mesh onto itself; a field with rho, U, W, E even and V odd in y stays so
    n = (6, 16, 5)
    gr = _channel_grid(n)
    gas = O.make_gas(mu=1 / 3000, mu_law=1, T_ref=CH["T_w"], omega=0.7, prandtl=0.7, T_wall=CH["T_w"])
    q, _ = inputs.channel(n)
    qs = 0.5 * (q + q[:, :, ::-1, :] * np.array([1, 1, -1, 1, 1])[:, None, None, None])
    q2, _ = O.run(gas, qs, None, 2, dt_fixed=2e-3, grid=gr)
    mirror = q2[:, :, ::-1, :] * np.array([1, 1, -1, 1, 1])[:, None, None, None]
    for v in range(5):
        assert np.abs(q2[v] - mirror[v]).max() <= 1e-13 * max(np.abs(q2[v]).max(), 1.0), v


def test_channel_inputs_decomposition_independent():
    full, _ = inputs.channel((8, 12, 10))
    part, _ = inputs.channel((8, 12, 10), z_begin=4, nz_local=3)
    np.testing.assert_array_equal(full[:, 4:7], part)
    T = (0.4 * (full[4] - 0.5 * (full[1] ** 2 + full[2] ** 2 + full[3] ** 2) / full[0])) / full[0]
    np.testing.assert_allclose(T, CH["T_w"], rtol=1e-13)


@pytest.mark.parametrize("vel", [(0.3, 0.0, 0.0), (0.2, -0.7, 0.1), (0.0, 0.0, 0.0)])
def test_cfl_dt_on_stretched_mesh_closed_form(vel):
    """O-13 + O-18 (stretched branch of or_cfl_dt): for a UNIFORM state the CFL step has the closed
    form dt = cfl * min_d min_j w_{d,j} / (|U_d| + c), c = sqrt(gamma p / rho), with the tanh cell
    widths w_{y,j} computed here from the face map of P:945-956 written out independently."""
    n = (12, 40, 10)
    gr = _channel_grid(n)
    rho, p = 1.3, 0.9
    q = np.zeros((5, n[2], n[1], n[0]))
    q[0] = rho
    for d in range(3):
        q[1 + d] = rho * vel[d]
    q[4] = p / 0.4 + 0.5 * rho * sum(v * v for v in vel)
    c = math.sqrt(1.4 * p / rho)
    b = 2.0
    yf = np.array([np.tanh(b * (2.0 * j / n[1] - 1.0)) / np.tanh(b) for j in range(n[1] + 1)])
    widths = [np.full(n[0], 2 * math.pi / n[0]), np.diff(yf), np.full(n[2], math.pi / n[2])]
    expect = 0.4 * min(widths[d].min() / (abs(vel[d]) + c) for d in range(3))
    got = O.cfl_dt(O.make_gas(T_wall=1.0), q, None, 0.4, grid=gr)
    assert got == pytest.approx(expect, rel=1e-13)
    # the wall cells are the narrowest: with V = 0 the y term wins only if it beats x and z
    assert widths[1].min() == pytest.approx(yf[1] - yf[0], rel=1e-14)
