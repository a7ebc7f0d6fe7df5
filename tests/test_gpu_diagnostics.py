"""GPU parity of the on-device volume diagnostics (hgks_diagnostics) against
the oracle's or_diagnostics on the same state (taken back with hgks_get_state, so fp32 runs compare
on identical inputs).  Both sides compute in fp64 and differ only in summation order: the oracle
sums cell by cell, whose error bound is (ncell - 1) u sum|x_i| (u = 2^-53), the GPU uses a tree.
Tolerance: ncell * u relative to the sum of magnitudes -- for the sign-definite entries that is
the value itself; eps_d (zero on the TGV initial field) is held to the eps_s scale, momenta
(zero by symmetry) to mass x rms velocity.  fp32 contexts store the wall-mirror ghosts in fp32
(the oracle mirrors the same fp32 interior in fp64), so with walls the bound is the fp32 unit
roundoff 2^-24."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs

pytestmark = pytest.mark.gpu

CH = inputs.channel_params()


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    H.lib()


def _compare(got, ref, ncell, mu, tol=None):
    tol = tol if tol is not None else max(ncell, 64) * 2.0 ** -53
    scale = np.abs(ref).copy()
    scale[3] = max(scale[3], scale[2])  # eps_d against the eps_s scale
    scale[5:8] = ref[4] * math.sqrt(2 * ref[0])  # momenta against mass x rms velocity
    # pressure-dilatation against its Cauchy-Schwarz bound mean(p) rms(div U), rms(div U)^2 =
    # (3/4) eps_d / mu (rho0 = 1), held to the eps_s-scale divergence when div U ~ 0 (TGV)
    rms_div = math.sqrt(0.75 * max(ref[3], ref[2]) / mu)
    scale[10] = max(scale[10], 0.4 * ref[8] / ref[9] * rms_div)
    err = np.abs(got - ref) / np.maximum(scale, 1e-300)
    assert err.max() <= tol, dict(zip(H.DIAG_NAMES, err))


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_tgv_diagnostics_parity(precision):
    n = 32
    q, dx = inputs.tgv(n)
    prm = inputs.tgv_params()
    L = 2 * math.pi
    with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=prm["mu"], precision=precision) as s:
        s.set_state(q)
        for nstep in (0, 3):
            s.step(nstep)
            got = H.hgks_diagnostics(s.ctx, rho0=1.0)
            qs = s.get_state()
            ref = O.diagnostics(O.make_gas(mu=prm["mu"]), qs, (L / n,) * 3)
            _compare(got, ref, n ** 3, prm["mu"])
            again = H.hgks_diagnostics(s.ctx, rho0=1.0)
            np.testing.assert_array_equal(got, again)  # deterministic reduction


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_channel_diagnostics_parity(precision):
    """walls (mirror ghosts) + tanh-stretched y: metric at cell centres, physical volumes."""
    n = (16, 40, 12)
    q, _ = inputs.channel(n)
    with H.Solver(n, CH["lo"], CH["hi"], mu=CH["mu_w"], mu_law=H.HGKS_MU_POWER, T_ref=CH["T_w"], omega=CH["omega"],
                  prandtl=CH["prandtl"], T_wall=CH["T_w"], bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                  stretch=(H.HGKS_UNIFORM, H.HGKS_TANH, H.HGKS_UNIFORM), stretch_b=(0.0, CH["b_g"], 0.0),
                  precision=precision, cfl=0.4) as s:
        s.set_state(q)
        s.step(2)
        got = H.hgks_diagnostics(s.ctx, rho0=1.0)
        qs = s.get_state()
    gas = O.make_gas(mu=CH["mu_w"], mu_law=1, T_ref=CH["T_w"], omega=CH["omega"], prandtl=CH["prandtl"],
                     T_wall=CH["T_w"])
    gr = O.make_grid(n, (2 * math.pi / n[0], 0.0, math.pi / n[2]), bc=(0, 1, 0), stretch=(0, 1, 0), lo=CH["lo"],
                     hi=CH["hi"], stretch_b=(0, CH["b_g"], 0))
    ref = O.diagnostics(gas, qs, None, grid=gr)
    _compare(got, ref, n[0] * n[1] * n[2], CH["mu_w"], tol=2.0 ** -24 if precision == H.HGKS_FP32 else None)
    assert got[H.DIAG_NAMES.index("volume")] == pytest.approx(2 * math.pi * 2 * math.pi, rel=1e-13)


def test_tgv_conservation_and_decay_on_gpu():
    """10 CFL steps of TGV 32^3: mass, momentum and total energy are conserved by the
    finite-volume update (to rounding); kinetic energy decays (viscous, Re = 1600)."""
    n = 32
    q, _ = inputs.tgv(n)
    prm = inputs.tgv_params()
    with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=prm["mu"]) as s:
        s.set_state(q)
        d0 = H.hgks_diagnostics(s.ctx)
        s.step(10)
        d1 = H.hgks_diagnostics(s.ctx)
    i = {k: j for j, k in enumerate(H.DIAG_NAMES)}
    assert d1[i["mass"]] == pytest.approx(d0[i["mass"]], rel=1e-13)
    assert d1[i["energy"]] == pytest.approx(d0[i["energy"]], rel=1e-13)
    mom_scale = d0[i["mass"]]
    for k in ("mom_x", "mom_y", "mom_z"):
        assert abs(d1[i[k]] - d0[i[k]]) <= 1e-13 * mom_scale
    assert d1[i["E_k"]] < d0[i["E_k"]]


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_per_step_history_matches_oracle(precision):
    """NEXT-2 time histories: the diagnostics fused into the stage-1 update hold, for
    every step, the state at the START of the step.  Each row must match or_diagnostics of the state
    the GPU had there (read back step by step in a twin context), and (t, dt) the step's."""
    n = 32
    q, dx = inputs.tgv(n)
    prm = inputs.tgv_params()
    gas = O.make_gas(mu=prm["mu"])
    kw = dict(mu=prm["mu"], precision=precision, cfl=0.4)
    with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, **kw) as s, \
            H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, **kw) as twin:
        H.hgks_history_enable(s.ctx, 16, rho0=1.0)
        s.set_state(q)
        twin.set_state(q)
        s.step(6)
        s.step(4)
        rows = H.hgks_history_read(s.ctx, 16)
        assert rows.shape == (10, H.HIST_COLS)
        t = 0.0
        for r in range(10):
            qs = twin.get_state()
            ref = O.diagnostics(gas, qs, (2 * math.pi / n,) * 3)
            _compare(rows[r, 2:], ref, n ** 3, prm["mu"])
            assert rows[r, 0] == t
            dt = twin.step(1)
            assert rows[r, 1] == dt
            t = twin.t
        np.testing.assert_array_equal(twin.get_state(), s.get_state())  # the history does not touch the step
        assert H.hgks_history_read(s.ctx, 16).shape[0] == 0
        with pytest.raises(H.HgksError):  # would overflow the 16 rows
            s.step(17)
