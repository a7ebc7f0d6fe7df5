"""Host post-processing of the channel plane statistics (paper_2207_01173_b200/channel_stats.py,
reading O-28) against closed forms: the laminar parabola has tau_w = 3 mu U_b / H exactly (the
wall fit is a quadratic), no fluctuations, and U_VD+ = U+ at uniform density; prescribed second
moments give the rms, Reynolds-stress and M_t values they encode."""
import math

import numpy as np
import pytest

from paper_2207_01173_b200 import channel_stats as CS
from paper_2207_01173_b200 import inputs

S = {k: i for i, k in enumerate(CS.STAT_NAMES)}
GAMMA = 1.4


def _plane_means(y, rho, U, p, V=None, UU_extra=0.0, VV_extra=0.0, UV_extra=0.0):
    ny = y.size
    V = np.zeros(ny) if V is None else V
    m = np.zeros((ny, len(CS.STAT_NAMES)))
    c = np.sqrt(GAMMA * p / rho)
    m[:, S["rho"]], m[:, S["U"]], m[:, S["V"]] = rho, U, V
    m[:, S["UU"]] = U * U + UU_extra
    m[:, S["VV"]] = V * V + VV_extra
    m[:, S["UV"]] = U * V + UV_extra
    m[:, S["rhoU"]], m[:, S["rhoV"]] = rho * U, rho * V
    m[:, S["rhoUV"]] = rho * (U * V + UV_extra)
    m[:, S["c"]], m[:, S["M"]], m[:, S["MM"]] = c, np.abs(U) / c, U * U / c ** 2
    m[:, S["T"]], m[:, S["p"]] = p / rho, p
    return m


@pytest.mark.parametrize("stretched", [False, True])
def test_laminar_parabola(stretched):
    ny, mu, Tw = 32, 1 / 3000, 2.857
    yf = inputs.tanh_faces(ny, -1, 1, 2.0) if stretched else np.linspace(-1, 1, ny + 1)
    y = 0.5 * (yf[1:] + yf[:-1])
    U = 1.5 * (1 - y * y)
    st = CS.ChannelStats(y, mu, Tw)
    for _ in range(3):
        st.add(_plane_means(y, np.ones(ny), U, np.full(ny, Tw)))
    pr = st.profiles()
    assert pr["tau_w"] == pytest.approx(3 * mu, rel=1e-12)
    assert pr["rho_w"] == pytest.approx(1.0, rel=1e-14)
    u_tau = math.sqrt(3 * mu)
    np.testing.assert_allclose(pr["U_plus"], U[: ny // 2] / u_tau, rtol=1e-12)
    np.testing.assert_allclose(pr["U_vd_plus"], pr["U_plus"], rtol=1e-12)
    np.testing.assert_allclose(pr["y_plus"], (y[: ny // 2] + 1) * u_tau / mu, rtol=1e-12)
    assert pr["Re_tau"] == pytest.approx(u_tau / mu, rel=1e-12)
    # rms = sqrt(<U^2> - <U>^2): the difference of raw moments carries ~eps <U>^2, so the floor is
    # sqrt(eps) |U+|, not eps
    floor = 4 * math.sqrt(2.0 ** -52) * pr["U_plus"].max()
    for k in ("u_rms_plus", "v_rms_plus", "w_rms_plus"):
        assert np.abs(pr[k]).max() <= floor, k
    assert np.abs(pr["M_t"]).max() <= 4 * math.sqrt(2.0 ** -52) * 1.5 / math.sqrt(GAMMA * Tw)
    assert np.abs(pr["reynolds_stress"]).max() <= 1e-12


def test_prescribed_fluctuations():
    ny, mu, Tw = 16, 0.01, 2.0
    y = inputs.cell_centres(ny, -1, 1)
    U = 1.5 * (1 - y * y)
    su, sv = 0.05, 0.03
    r = 0.01 * y  # <U'V'>: negative in the lower half, antisymmetric
    st = CS.ChannelStats(y, mu, Tw)
    st.add(_plane_means(y, np.ones(ny), U, np.full(ny, Tw), UU_extra=su ** 2, VV_extra=sv ** 2, UV_extra=r))
    pr = st.profiles()
    u_tau, tau = pr["u_tau"], pr["tau_w"]
    np.testing.assert_allclose(pr["u_rms_plus"], su / u_tau, rtol=1e-10)
    np.testing.assert_allclose(pr["v_rms_plus"], sv / u_tau, rtol=1e-10)
    np.testing.assert_allclose(pr["reynolds_stress"], -0.01 * y[: ny // 2] / tau, rtol=1e-10)
    c = math.sqrt(GAMMA * Tw)
    np.testing.assert_allclose(pr["M_t"], math.sqrt(su ** 2 + sv ** 2) / c, rtol=1e-10)


def test_van_driest_density_weighting():
    """<rho> = 4 rho_w off the wall: the trapezoid weight is (1 + 2)/2 on the first interval and 2 after."""
    ny, mu, Tw = 16, 0.01, 2.0
    y = inputs.cell_centres(ny, -1, 1)
    U = 1.5 * (1 - y * y)
    rho = np.full(ny, 4.0)
    p = np.full(ny, Tw)       # rho_w = p / T_w = 1
    st = CS.ChannelStats(y, mu, Tw)
    st.add(_plane_means(y, rho, U, p))
    pr = st.profiles()
    Up = pr["U_plus"]
    np.testing.assert_allclose(pr["U_vd_plus"], 1.5 * Up[0] + 2.0 * (Up - Up[0]), rtol=1e-12)


def test_shape_check():
    st = CS.ChannelStats(np.zeros(4), 1.0, 1.0)
    with pytest.raises(ValueError):
        st.add(np.zeros((5, 16)))
