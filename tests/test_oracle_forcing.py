"""Pins of the oracle's streamwise body force (or_run_forced, readings O-26, O-27)
against closed forms:

* uniform flow under a constant acceleration f: the flux divergence vanishes, the source is
  (0, rho f, 0, 0, rho U f) and its time derivative (0, 0, 0, 0, rho f^2) is constant, so S2O4
  integrates it exactly: rho U = rho (U0 + f t), p unchanged.
* dead-beat controller (mode 2) in a drag-free periodic box: f^0 = (m_b - m^0)/(dt rho_b) puts the
  bulk momentum on target in one step, after which f = 0.
* laminar Poiseuille channel: at steady state the force balances the wall shear,
  f rho_b = tau_w / H with tau_w = 3 mu U_b / H, i.e. f = 3 mu U_b / (rho_b H^2); the controller's
  transient from f_init = 0 is f^1 = 2W, f^n = W (W = drag per unit mass) by its definition.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_01173_b200 import inputs

GAMMA = 1.4


def _uniform(n, rho, U, p):
    return inputs.uniform(n, rho=rho, vel=U, p=p)


def test_constant_acceleration_uniform_flow_is_exact():
    n = (6, 6, 6)
    rho, U0, p, f, dt, steps = 1.3, (0.2, -0.1, 0.05), 1.0, 0.3, 0.01, 7
    q = _uniform(n, rho, U0, p)
    q1, _, fh = O.run_forced(O.make_gas(mu=0.01), q, (0.5, 0.5, 0.5), steps, mode=1, force=f, dt_fixed=dt)
    t = steps * dt
    U = (U0[0] + f * t, U0[1], U0[2])
    ref = inputs.prim_to_cons(np.full(n[::-1], rho), *U, p)
    np.testing.assert_allclose(q1, ref, rtol=1e-14, atol=1e-15)
    assert np.all(fh == f)


def test_deadbeat_reaches_target_in_one_step():
    n = (6, 6, 6)
    rho, dt = 1.3, 0.02
    q = _uniform(n, rho, (0.2, 0.0, 0.0), 1.0)
    target = rho * 0.5
    q1, _, fh = O.run_forced(O.make_gas(mu=0.01), q, (0.5, 0.5, 0.5), 4, mode=2, force=0.0, target=target,
                             dt_fixed=dt)
    f0 = (target - rho * 0.2) / (dt * rho)
    assert fh[0] == pytest.approx(f0, rel=1e-13)
    assert np.abs(fh[1:]).max() <= 1e-12 * f0
    assert (q1[1] / q1[0]).mean() == pytest.approx(0.5, rel=1e-13)


def test_laminar_poiseuille_force_balance():
    """walls at y = -1, 1 (uniform y, H = 1), rho_b = 2, U = 1.5 U_b (1 - y^2), Ma 0.1, mu 0.02
    (Re_b = 100), bulk target = the initial bulk: f -> 3 mu U_b / rho_b to the scheme's O(h^2)
    wall-shear error (1% bound; measured 0.3% at ny = 16), profile and bulk held."""
    ny, nx, nz = 16, 5, 5
    Ma, mu, rho = 0.1, 0.02, 2.0
    Tw = 1.0 / (GAMMA * Ma * Ma)
    gas = O.make_gas(mu=mu, prandtl=0.7, T_wall=Tw)
    gr = O.make_grid((nx, ny, nz), (2 * math.pi / nx, 2.0 / ny, math.pi / nz), bc=(0, 1, 0), lo=(0, -1, 0),
                     hi=(2 * math.pi, 1, math.pi))
    y = inputs.cell_centres(ny, -1, 1)
    U = np.broadcast_to((1.5 * (1 - y ** 2))[None, :, None], (nz, ny, nx))
    q = inputs.prim_to_cons(np.full(U.shape, rho), U, 0 * U, 0 * U, rho * Tw)
    m0 = float(q[1].mean())
    q1, _, fh = O.run_forced(gas, q, None, 60, mode=2, force=0.0, target=m0, grid=gr)
    f_bal = 3 * mu * 1.0 / rho
    assert fh[-1] == pytest.approx(f_bal, rel=1e-2)
    assert fh[1] == pytest.approx(2 * fh[2], rel=1e-2)      # f^1 = 2W, f^2 = W
    assert q1[1].mean() == pytest.approx(m0, rel=1e-6)
    Un = q1[1] / q1[0]
    assert np.abs(Un - U).max() <= 1e-3 * 1.5
