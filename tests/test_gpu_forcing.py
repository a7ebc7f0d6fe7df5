"""GPU parity of the streamwise body force (readings O-26 source, O-27 dead-beat bulk controller;
SURVEY §8(f) NEXT-1) against the oracle's or_run_forced, through the C ABI.  Tolerances as in
test_gpu_parity.py (fp64 1e-11 normwise, fp32 1e-4), force histories fp64 rel 1e-9 (the force is
a difference quotient (m_b - m)/dt of bulk sums, amplifying their rounding by 1/dt)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs
from tests import diagnostics as D

pytestmark = pytest.mark.gpu

CH = inputs.channel_params()


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    H.lib()


def test_constant_acceleration_uniform_flow_exact():
    n = (6, 6, 6)
    rho, U0, p, f, dt, steps = 1.3, (0.2, -0.1, 0.05), 1.0, 0.3, 0.01, 7
    q = inputs.uniform(n, rho=rho, vel=U0, p=p)
    with H.Solver(n, (0, 0, 0), (3, 3, 3), mu=0.01, dt_fixed=dt, force_mode=H.HGKS_FORCE_CONST, force=f) as s:
        s.set_state(q)
        s.step(steps)
        got = s.get_state()
        assert H.hgks_get_forcing(s.ctx)[0] == f
    ref = inputs.prim_to_cons(np.full(n[::-1], rho), U0[0] + f * steps * dt, U0[1], U0[2], p)
    np.testing.assert_allclose(got, ref, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_deadbeat_periodic_box(precision):
    n = (6, 6, 6)
    rho, dt = 1.3, 0.02
    q = inputs.uniform(n, rho=rho, vel=(0.2, 0.0, 0.0), p=1.0)
    target = rho * 0.5
    fo = []
    with H.Solver(n, (0, 0, 0), (3, 3, 3), mu=0.01, dt_fixed=dt, force_mode=H.HGKS_FORCE_BULK, force=0.0,
                  force_target=target, precision=precision) as s:
        s.set_state(q)
        for _ in range(3):
            s.step(1)
            fo.append(H.hgks_get_forcing(s.ctx))
        got = s.get_state()
    f0 = (target - rho * 0.2) / (dt * rho)
    tol = 1e-12 if precision == H.HGKS_FP64 else 1e-5
    assert fo[0][0] == pytest.approx(f0, rel=tol)
    assert abs(fo[1][0]) <= (1e-10 if precision == H.HGKS_FP64 else 1e-3) * f0
    assert fo[-1][1] == pytest.approx(target, rel=tol) and fo[-1][2] == pytest.approx(rho, rel=tol)
    assert (got[1] / got[0]).mean() == pytest.approx(0.5, rel=tol)


def _laminar(ny=16):
    Ma, mu, rho = 0.1, 0.02, 2.0
    Tw = 1.0 / (1.4 * Ma * Ma)
    n = (5, ny, 5)
    y = inputs.cell_centres(ny, -1, 1)
    U = np.broadcast_to((1.5 * (1 - y ** 2))[None, :, None], n[::-1])
    q = np.ascontiguousarray(inputs.prim_to_cons(np.full(U.shape, rho), U, 0 * U, 0 * U, rho * Tw))
    return n, q, mu, Tw


def test_laminar_poiseuille_parity_and_balance():
    """walls in y, uniform mesh, 40 CFL steps with the bulk controller: state and force history
    match the oracle; the force settles on the wall-shear balance 3 mu U_b / rho_b."""
    n, q, mu, Tw = _laminar()
    m0 = float(q[1].mean())
    lo, hi = (0, -1, 0), (2 * math.pi, 1, math.pi)
    steps = 40
    fg = []
    with H.Solver(n, lo, hi, mu=mu, prandtl=0.7, T_wall=Tw, bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                  force_mode=H.HGKS_FORCE_BULK, force=0.0, force_target=m0) as s:
        s.set_state(q)
        for _ in range(steps):
            s.step(1)
            fg.append(H.hgks_get_forcing(s.ctx)[0])
        got = s.get_state()
    gas = O.make_gas(mu=mu, prandtl=0.7, T_wall=Tw)
    gr = O.make_grid(n, (2 * math.pi / n[0], 2.0 / n[1], math.pi / n[2]), bc=(0, 1, 0), lo=lo, hi=hi)
    qo, _, fo = O.run_forced(gas, q, None, steps, mode=2, force=0.0, target=m0, grid=gr)
    assert D.normwise_error(got, qo).max() <= 1e-11
    fg = np.array(fg)
    assert np.abs(fg[1:] - fo[1:]).max() <= 1e-9 * np.abs(fo[1:]).max()
    assert fg[-1] == pytest.approx(3 * mu / 2.0, rel=1e-2)


@pytest.mark.parametrize("precision,tol", [(H.HGKS_FP64, 1e-11), (H.HGKS_FP32, 1e-4)])
def test_channel_config4_forced_parity(precision, tol):
    """BASELINE config 4 physics (tanh y, power-law mu, Pr 0.7, isothermal walls) at 32 x 64 x 32 with
    the bulk controller holding the initial bulk momentum, 8 CFL steps, against the oracle."""
    n = (32, 64, 32)
    q, _ = inputs.channel(n)
    gas = O.make_gas(mu=CH["mu_w"], mu_law=1, T_ref=CH["T_w"], omega=CH["omega"], prandtl=CH["prandtl"],
                     T_wall=CH["T_w"])
    gr = O.make_grid(n, (2 * math.pi / n[0], 0.0, math.pi / n[2]), bc=(0, 1, 0), stretch=(0, 1, 0), lo=CH["lo"],
                     hi=CH["hi"], stretch_b=(0, CH["b_g"], 0))
    target = float(O.diagnostics(gas, q, None, grid=gr)[5] / O.diagnostics(gas, q, None, grid=gr)[9])
    steps = 8
    with H.Solver(n, CH["lo"], CH["hi"], mu=CH["mu_w"], mu_law=H.HGKS_MU_POWER, T_ref=CH["T_w"], omega=CH["omega"],
                  prandtl=CH["prandtl"], T_wall=CH["T_w"], bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                  stretch=(H.HGKS_UNIFORM, H.HGKS_TANH, H.HGKS_UNIFORM), stretch_b=(0.0, CH["b_g"], 0.0),
                  precision=precision, force_mode=H.HGKS_FORCE_BULK, force=0.0, force_target=target) as s:
        s.set_state(q)
        s.step(steps)
        got = s.get_state()
        f_last, m_last, _ = H.hgks_get_forcing(s.ctx)
    qo, _, fo = O.run_forced(gas, q, None, steps, mode=2, force=0.0, target=target, grid=gr)
    assert D.normwise_error(got, qo).max() <= tol
    assert m_last == pytest.approx(target, rel=1e-9 if precision == H.HGKS_FP64 else 1e-5)
    if precision == H.HGKS_FP64:
        assert f_last == pytest.approx(fo[-1], rel=1e-6)
