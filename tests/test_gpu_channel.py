"""GPU parity of the channel configuration (BASELINE config 4): isothermal no-slip
walls in y (O-17), tanh-stretched y (O-18), mu = mu_w (T/T_w)^0.7 and the Pr = 0.7 heat-flux fix
(O-12), through the C ABI against the oracle.  Tolerances as in test_gpu_parity.py."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs
from tests import diagnostics as D
from tests.test_gpu_parity import _oracle_records, _random_records, _rowwise

pytestmark = pytest.mark.gpu

CH = inputs.channel_params()
LO, HI = CH["lo"], CH["hi"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    H.lib()


def _gas():
    return O.make_gas(mu=CH["mu_w"], mu_law=1, T_ref=CH["T_w"], omega=CH["omega"], prandtl=CH["prandtl"],
                      T_wall=CH["T_w"])


def _grid(n):
    return O.make_grid(n, (2 * math.pi / n[0], 0.0, math.pi / n[2]), bc=(0, 1, 0), stretch=(0, 1, 0), lo=LO, hi=HI,
                       stretch_b=(0, CH["b_g"], 0))


def _solver(n, **kw):
    kw.setdefault("cfl", 0.4)
    return H.Solver(n, LO, HI, mu=CH["mu_w"], mu_law=H.HGKS_MU_POWER, T_ref=CH["T_w"], omega=CH["omega"],
                    prandtl=CH["prandtl"], T_wall=CH["T_w"], bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                    stretch=(H.HGKS_UNIFORM, H.HGKS_TANH, H.HGKS_UNIFORM), stretch_b=(0.0, CH["b_g"], 0.0), **kw)


@pytest.mark.parametrize("precision,tf,tdf", [(H.HGKS_FP64, 1e-13, 1e-11), (H.HGKS_FP32, 2e-5, 1e-3)])
def test_gp_flux_parity_power_law_prandtl(precision, tf, tdf):
    rec = _random_records(300, seed=31, pscale=CH["T_w"], gscale=0.5)
    kw = dict(mu=CH["mu_w"], mu_law=1, T_ref=CH["T_w"], omega=CH["omega"], prandtl=CH["prandtl"])
    got = H.hgks_test_gp_flux(rec, 2e-3, precision=precision, **kw)
    ref = _oracle_records(rec, 2e-3, None, gas=O.make_gas(**kw))
    assert _rowwise(got[:, :5], ref[:, :5]).max() <= tf
    assert _rowwise(got[:, 5:10], ref[:, 5:10]).max() <= tdf


def test_operator_parity_channel_ragged():
    n = (12, 22, 10)
    q, _ = inputs.channel(n)
    dt = 2e-3
    with _solver(n, dt_fixed=dt) as s:
        s.set_state(q)
        L, dL = H.hgks_test_operator(s.ctx, dt, q.shape)
    Lo, dLo = O.operator(_gas(), q, None, dt, grid=_grid(n))
    assert D.normwise_error(q + dt * L, q + dt * Lo).max() <= 1e-14
    assert D.normwise_error(q + dt * dt * dL, q + dt * dt * dLo).max() <= 1e-14
    assert D.normwise_error(L, Lo).max() <= 1e-10


@pytest.mark.parametrize("precision,tol", [(H.HGKS_FP64, 1e-11), (H.HGKS_FP32, 1e-4)])
def test_step_parity_channel_reduced_config4(precision, tol):
    # BASELINE config 4 at reduced size 32 x 64 x 32, 10 CFL steps
    n = (32, 64, 32)
    q, _ = inputs.channel(n)
    gas, gr = _gas(), _grid(n)
    g_states, g_dts = [], []
    with _solver(n, precision=precision) as s:
        s.set_state(q)
        for _ in range(10):
            g_dts.append(s.step(1))
            g_states.append(s.get_state())
    qo = q
    for k in range(10):
        qo, hist = O.run(gas, qo, None, 1, grid=gr)
        assert g_dts[k] == pytest.approx(hist[0], rel=1e-13 if precision == H.HGKS_FP64 else 1e-6)
        e = D.normwise_error(g_states[k], qo)
        assert e.max() <= tol, (k, e)
        assert abs(D.kinetic_energy(g_states[k]) - D.kinetic_energy(qo)) <= tol * D.kinetic_energy(qo)


def test_rest_state_between_walls_bitwise():
    n = (8, 16, 6)
    q = inputs.uniform(n, rho=1.3, vel=(0.0, 0.0, 0.0), p=1.3 * CH["T_w"])
    with _solver(n, dt_fixed=1e-3) as s:
        s.set_state(q)
        q0 = s.get_state()
        s.step(3)
        np.testing.assert_array_equal(s.get_state(), q0)


def _oracle_column_step(q, n, dt, ci, ck):
    """Exact oracle value of one S2O4 step on the full y column (ci, ck) of the channel, from the
    13 x ny x 13 neighbourhood: periodic x/z data cut from the field (bc 2 = ghosts supplied), wall
    ghosts in y filled by the oracle."""
    nx, ny, nz = n
    gas = _gas()
    xs = (np.arange(-6, 7) + ci) % nx
    zs = (np.arange(-6, 7) + ck) % nz
    blk = np.zeros((5, 13, ny + 6, 13))
    blk[:, :, 3:-3, :] = q[:, zs][:, :, :, xs]
    g1 = O.make_grid((7, ny, 7), (2 * math.pi / nx, 0.0, math.pi / nz), bc=(2, 1, 2), stretch=(0, 1, 0), lo=LO, hi=HI,
                     stretch_b=(0, CH["b_g"], 0))
    O.lib().or_fill_ghosts(O.C.byref(gas), O.C.byref(g1), O._p(blk))
    L, dL = O.operator(gas, np.zeros((5, 7, ny, 7)), None, dt, qg=blk, grid=g1)
    inner = np.ascontiguousarray(blk[:, 3:10, 3:-3, 3:10])
    qs = O.s2o4_stage1(inner, L, dL, dt)
    blk2 = np.zeros((5, 7, ny + 6, 7))
    blk2[:, :, 3:-3, :] = qs
    g2 = O.make_grid((1, ny, 1), (2 * math.pi / nx, 0.0, math.pi / nz), bc=(2, 1, 2), stretch=(0, 1, 0), lo=LO, hi=HI,
                     stretch_b=(0, CH["b_g"], 0))
    O.lib().or_fill_ghosts(O.C.byref(gas), O.C.byref(g2), O._p(blk2))
    Ls, dLs = O.operator(gas, np.zeros((5, 1, ny, 1)), None, dt, qg=blk2, grid=g2)
    c = (slice(None), slice(3, 4), slice(None), slice(3, 4))
    return O.s2o4_final(np.ascontiguousarray(inner[c]), np.ascontiguousarray(L[c]), np.ascontiguousarray(dL[c]), dLs, dt)[:, 0, :, 0]


@pytest.mark.parametrize("precision,tol", [(H.HGKS_FP64, 1e-11), (H.HGKS_FP32, 1e-4)])
def test_full_size_h2_sampled_columns(precision, tol):
    """Config 4 full size (H2: 128 x 256 x 128), one CFL step; three full wall-to-wall columns
    against the oracle's exact local evaluation."""
    n = (128, 256, 128)
    q, _ = inputs.channel(n)
    with _solver(n, precision=precision) as s:
        s.set_state(q)
        dt = s.step(1)
        q1 = s.get_state()
    dt_o = O.cfl_dt(_gas(), q, None, 0.4, grid=_grid(n))
    assert dt == pytest.approx(dt_o, rel=1e-13 if precision == H.HGKS_FP64 else 1e-6)
    mom = np.sqrt((q1[1:4] ** 2).sum(0)).max()
    den = np.array([np.abs(q1[0]).max(), mom, mom, mom, np.abs(q1[4]).max()])
    for ci, ck in ((0, 0), (77, 5), (127, 126)):
        ref = _oracle_column_step(q, n, dt_o, ci, ck)
        got = q1[:, ck, :, ci]
        err = (np.abs(got - ref).max(axis=1) / den).max()
        assert err <= tol, (ci, ck, err)
