"""Channel physics on the GPU: the x-z plane statistics reduction against the
oracle, and the laminar channel validation -- a plug flow between isothermal no-slip walls driven
by the bulk-momentum controller (O-27) must converge to the analytic Poiseuille profile
U = 1.5 U_b (1 - y^2) and the force to the wall-shear balance f = 3 mu U_b / (rho_b H^2)
(within 1% L-infinity and 1%).  ~4e4 steps: GPU only."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_01173_b200 import channel_stats as CS
from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs

pytestmark = pytest.mark.gpu

CH = inputs.channel_params()


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    H.lib()


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_plane_stats_parity(precision):
    n = (16, 40, 12)
    q, _ = inputs.channel(n)
    with H.Solver(n, CH["lo"], CH["hi"], mu=CH["mu_w"], mu_law=H.HGKS_MU_POWER, T_ref=CH["T_w"], omega=CH["omega"],
                  prandtl=CH["prandtl"], T_wall=CH["T_w"], bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                  stretch=(H.HGKS_UNIFORM, H.HGKS_TANH, H.HGKS_UNIFORM), stretch_b=(0.0, CH["b_g"], 0.0),
                  precision=precision) as s:
        s.set_state(q)
        s.step(2)
        got = s.plane_stats()
        again = s.plane_stats()
        qs = s.get_state()
    ref = O.plane_stats(O.make_gas(), qs, (1.0, 1.0, 1.0))
    np.testing.assert_array_equal(got, again)
    # summation order only: n_plane * eps relative to the mean magnitude of each moment
    scale = np.maximum(np.abs(ref), np.abs(ref).max(axis=0, keepdims=True) * 1e-3)
    assert (np.abs(got - ref) / scale).max() <= n[0] * n[2] * 2.0 ** -53 * 4


def test_laminar_channel_converges_to_poiseuille():
    ny, mu, Ma, rho_b, U_b = 32, 0.1, 0.05, 1.0, 1.0
    Tw = 1.0 / (1.4 * Ma * Ma)
    n = (5, ny, 5)
    lo, hi = (0.0, -1.0, 0.0), (2 * math.pi, 1.0, math.pi)
    shape = n[::-1]
    q = inputs.prim_to_cons(np.full(shape, rho_b), np.full(shape, U_b), 0.0, 0.0, rho_b * Tw)
    steps = 40000  # t ~ 50 = 5 H^2/nu: slowest mode decayed by exp(-pi^2/4 * 5) ~ 4e-6
    with H.Solver(n, lo, hi, mu=mu, prandtl=0.7, T_wall=Tw, bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                  force_mode=H.HGKS_FORCE_BULK, force=0.0, force_target=rho_b * U_b) as s:
        s.set_state(q)
        s.step(steps)
        assert s.t > 45.0
        f, m, rb = H.hgks_get_forcing(s.ctx)
        pm = s.plane_stats()
        # a t_end-clamped step changes dt abruptly: the dead-beat law then misses by O(dt * delta dt)
        # (the flux time derivative does not see the force, O-26), and recovers on the next steps
        s.step(10, t_end=s.t + 0.6 * 1.2e-3)
        m_clamped = H.hgks_get_forcing(s.ctx)[1]
        s.step(5)
        m_after = H.hgks_get_forcing(s.ctx)[1]
    assert abs(m_clamped - rho_b * U_b) <= 1e-5
    assert abs(m_after - rho_b * U_b) <= 1e-6
    y = inputs.cell_centres(ny, -1, 1)
    U = pm[:, CS.STAT_NAMES.index("U")]
    exact = 1.5 * U_b * (1 - y * y)
    # the finite-volume state holds cell averages: compare with the parabola's cell averages
    h = 2.0 / ny
    exact_avg = exact - 1.5 * U_b * h * h / 12
    assert np.abs(U - exact_avg).max() <= 1e-2 * 1.5 * U_b
    assert m == pytest.approx(rho_b * U_b, rel=1e-9)
    assert f == pytest.approx(3 * mu * U_b / rb, rel=1e-2)
    st = CS.ChannelStats(y, mu, Tw)
    st.add(pm)
    pr = st.profiles()
    assert pr["tau_w"] == pytest.approx(3 * mu * U_b, rel=2e-2)
    assert pr["u_rms_plus"].max() < 1e-4
