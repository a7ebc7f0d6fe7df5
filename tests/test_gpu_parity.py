"""GPU parity: the CUDA path (through the C ABI, include/hgks.h + hgks_test.h) against the oracle
on identical seeded inputs.  Tolerances (BASELINE north_star):
  fp64: normwise (O-19) <= 1e-11 on conservative variables after 10 steps, and per-step E_k and
        enstrophy relative <= 1e-11;  per-piece checks (Gauss-point flux, operator) tighter;
  fp32: <= 1e-4 with the same metric, against the fp64 oracle.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs
from tests import diagnostics as D

pytestmark = pytest.mark.gpu

TGV = inputs.tgv_params()
TWO_PI = 2 * math.pi


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device (no CPU fallback exists)"
    H.lib()


def _solver(n, lo, hi, **kw):
    return H.Solver(n, lo, hi, **kw)


def _tgv_solver(n, **kw):
    kw.setdefault("mu", TGV["mu"])
    return _solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, **kw)


def _prim_to_cons(rho, U, V, W, p, gamma=1.4):
    return np.array([rho, rho * U, rho * V, rho * W, p / (gamma - 1) + 0.5 * rho * (U * U + V * V + W * W)])


def _random_records(n, seed, pscale=1.0, gscale=0.3):
    rng = np.random.default_rng(seed)
    rec = np.zeros((n, 55))
    for r in range(n):
        pl = np.array([rng.uniform(0.5, 2.0), *rng.normal(scale=0.6, size=3), pscale * rng.uniform(0.5, 3.0)])
        pr = pl.copy()
        pr[0] *= 1 + rng.normal(scale=0.05)
        pr[4] *= 1 + rng.normal(scale=0.05)
        pr[1:4] += rng.normal(scale=0.1, size=3)
        if r % 7 == 0:
            pl[1] = pr[1] = 0.0  # stagnation: exercises erfc(0)
        Wl, Wr = _prim_to_cons(*pl), _prim_to_cons(*pr)
        sc = np.abs(Wl) + 0.1
        rec[r, 0:5] = Wl
        rec[r, 5:10] = Wr
        rec[r, 10:55] = (rng.normal(scale=gscale, size=(9, 5)) * sc).ravel()
    return rec


def _oracle_records(rec, dt, mu, gas=None):  # noqa: D103
    gas = gas or O.make_gas(mu=mu)
    out = np.zeros((rec.shape[0], 11))
    for r in range(rec.shape[0]):
        x = rec[r]
        F, dF, tau = O.gp_flux(gas, x[0:5], x[10:25].reshape(3, 5), x[5:10], x[25:40].reshape(3, 5),
                               x[40:55].reshape(3, 5), dt)
        out[r, :5], out[r, 5:10], out[r, 10] = F, dF, tau
    return out


def _rowwise(a, b):
    return np.abs(a - b).max(axis=1) / np.abs(b).max(axis=1)


@pytest.mark.parametrize("mu,dt", [(1e-3, 1e-2), (6.25e-4, 7.1e-3), (0.0, 1e-2), (0.05, 1e-2)])
def test_gp_flux_parity_fp64(mu, dt):
    rec = _random_records(400, seed=int(mu * 1e6) + 3)
    got = H.hgks_test_gp_flux(rec, dt, mu=mu)
    ref = _oracle_records(rec, dt, mu)
    assert _rowwise(got[:, :5], ref[:, :5]).max() <= 1e-13
    assert _rowwise(got[:, 5:10], ref[:, 5:10]).max() <= 1e-11
    np.testing.assert_allclose(got[:, 10], ref[:, 10], rtol=1e-14, atol=0)


def test_gp_flux_parity_tgv_scales():
    # TGV magnitudes: p ~ 71, tau/dt ~ 1e-3
    rec = _random_records(400, seed=9, pscale=71.0, gscale=1.0)
    got = H.hgks_test_gp_flux(rec, 7.149e-3, mu=TGV["mu"])
    ref = _oracle_records(rec, 7.149e-3, TGV["mu"])
    assert _rowwise(got[:, :5], ref[:, :5]).max() <= 1e-13
    assert _rowwise(got[:, 5:10], ref[:, 5:10]).max() <= 1e-11


def test_gp_flux_parity_fp32():
    rec = _random_records(400, seed=21)
    got = H.hgks_test_gp_flux(rec, 1e-2, mu=1e-3, precision=H.HGKS_FP32)
    ref = _oracle_records(rec, 1e-2, 1e-3)
    assert _rowwise(got[:, :5], ref[:, :5]).max() <= 2e-5
    assert _rowwise(got[:, 5:10], ref[:, 5:10]).max() <= 1e-3


def _operator_check(q, dx, lo, hi, mu, dt, precision=H.HGKS_FP64):
    """L, d_t L of one stage vs the oracle.  Face fluxes are O(|Q| c) while L is their small
    difference (the TGV energy flux ~250 vs d(rhoE)/dt ~ 1), so rounding differences are judged at
    the state level: dt |dL| and dt^2 |d(d_t L)| relative to max|Q_v| <= 1e-14 (momenta grouped),
    plus a gross-error bound relative to max|L| itself."""
    nz, ny, nx = q.shape[1:]
    with _solver((nx, ny, nz), lo, hi, mu=mu, dt_fixed=dt, precision=precision) as s:
        s.set_state(q)
        L, dL = H.hgks_test_operator(s.ctx, dt, q.shape)
    Lo, dLo = O.operator(O.make_gas(mu=mu), q, dx, dt)
    qn = D.normwise_error(q + dt * L, q + dt * Lo)
    qdn = D.normwise_error(q + dt * dt * dL, q + dt * dt * dLo)
    assert qn.max() <= 1e-14, qn
    assert qdn.max() <= 1e-14, qdn
    assert D.normwise_error(L, Lo).max() <= 1e-10
    assert D.normwise_error(dL, dLo).max() <= 1e-10


def test_operator_parity_ragged_perturbed():
    # several 8x8 tiles plus ragged tails on every axis
    q, dx = inputs.perturbed((21, 13, 11), seed=5, amp=0.08)
    hi = (dx[0] * 21, dx[1] * 13, dx[2] * 11)
    _operator_check(q, dx, (0, 0, 0), hi, 2e-3, 0.01)


def test_operator_parity_tgv16():
    q, dx = inputs.tgv(16)
    _operator_check(q, dx, (-math.pi,) * 3, (math.pi,) * 3, TGV["mu"], 0.0143)


def _run_gpu_steps(q, nsteps, n, lo, hi, **kw):
    states, dts = [], []
    with _solver(n, lo, hi, **kw) as s:
        s.set_state(q)
        for _ in range(nsteps):
            dts.append(s.step(1))
            states.append(s.get_state())
    return states, dts


def _run_oracle_steps(q, nsteps, dx, mu, dt_fixed=0.0):
    states, dts = [], []
    gas = O.make_gas(mu=mu)
    for _ in range(nsteps):
        q, h = O.run(gas, q, dx, 1, dt_fixed=dt_fixed)
        states.append(q)
        dts.append(h[0])
    return states, dts


def test_step_parity_tgv32_fp64_config1():
    # BASELINE config 1: TGV Re=1600 Ma=0.1, 32^3, 10 S2O4 steps, FP64, CFL mode (A0 included)
    q, dx = inputs.tgv(32)
    g_states, g_dts = _run_gpu_steps(q, 10, (32,) * 3, (-math.pi,) * 3, (math.pi,) * 3, mu=TGV["mu"], cfl=0.4)
    o_states, o_dts = _run_oracle_steps(q, 10, dx, TGV["mu"])
    np.testing.assert_allclose(g_dts, o_dts, rtol=1e-13)
    assert o_dts[0] == pytest.approx(7.14933e-3, rel=1e-5)  # SURVEY A.10 (CFL 0.4 on this field)
    for k, (a, b) in enumerate(zip(g_states, o_states)):
        e = D.normwise_error(a, b)
        assert e.max() <= 1e-11, (k, e)
        assert abs(D.kinetic_energy(a) - D.kinetic_energy(b)) <= 1e-11 * D.kinetic_energy(b)
        zb = D.enstrophy(b, dx)
        assert abs(D.enstrophy(a, dx) - zb) <= 1e-11 * zb


def test_step_parity_ragged_fixed_dt():
    q, dx = inputs.perturbed((21, 13, 11), seed=7, amp=0.08)
    hi = (dx[0] * 21, dx[1] * 13, dx[2] * 11)
    g_states, _ = _run_gpu_steps(q, 3, (21, 13, 11), (0, 0, 0), hi, mu=2e-3, dt_fixed=0.02)
    o_states, _ = _run_oracle_steps(q, 3, dx, 2e-3, dt_fixed=0.02)
    for a, b in zip(g_states, o_states):
        assert D.normwise_error(a, b).max() <= 1e-12


def test_step_parity_tgv32_fp32():
    # BASELINE fp32 tolerance 1e-4 (normwise, O-19) against the fp64 oracle after 10 steps
    q, dx = inputs.tgv(32)
    g_states, g_dts = _run_gpu_steps(q, 10, (32,) * 3, (-math.pi,) * 3, (math.pi,) * 3, mu=TGV["mu"],
                                     cfl=0.4, precision=H.HGKS_FP32)
    o_states, o_dts = _run_oracle_steps(q, 10, dx, TGV["mu"])
    np.testing.assert_allclose(g_dts, o_dts, rtol=1e-6)
    for k, (a, b) in enumerate(zip(g_states, o_states)):
        e = D.normwise_error(a, b)
        assert e.max() <= 1e-4, (k, e)
        assert abs(D.kinetic_energy(a) - D.kinetic_energy(b)) <= 1e-4 * D.kinetic_energy(b)
        zb = D.enstrophy(b, dx)
        assert abs(D.enstrophy(a, dx) - zb) <= 1e-4 * zb


def test_step_parity_tgv128_config2_fp64_and_fp32():
    """BASELINE config 2: TGV 128^3, FP64 and FP32 on one B200, 10 CFL steps against the FP64 oracle
    stepped alongside (~30 s of oracle time per step on 16 host cores): normwise (O-19) <= 1e-11 / 1e-4
    after every step, per-step E_k and enstrophy to the same tolerances, dt to 1e-13 / 1e-6."""
    n = 128
    q, dx = inputs.tgv(n)
    gas = O.make_gas(mu=TGV["mu"])
    tol = {H.HGKS_FP64: 1e-11, H.HGKS_FP32: 1e-4}
    dtol = {H.HGKS_FP64: 1e-13, H.HGKS_FP32: 1e-6}
    worst = {p: 0.0 for p in tol}
    with _tgv_solver(n, cfl=0.4) as s64, _tgv_solver(n, cfl=0.4, precision=H.HGKS_FP32) as s32:
        s64.set_state(q)
        s32.set_state(q)
        qo = q
        for k in range(10):
            qo, h = O.run(gas, qo, dx, 1)
            ko, zo = D.kinetic_energy(qo), D.enstrophy(qo, dx)
            for prec, s in ((H.HGKS_FP64, s64), (H.HGKS_FP32, s32)):
                dt = s.step(1)
                assert dt == pytest.approx(h[0], rel=dtol[prec]), (prec, k)
                a = s.get_state()
                e = D.normwise_error(a, qo).max()
                worst[prec] = max(worst[prec], e)
                assert e <= tol[prec], (prec, k, e)
                assert abs(D.kinetic_energy(a) - ko) <= tol[prec] * ko, (prec, k)
                assert abs(D.enstrophy(a, dx) - zo) <= tol[prec] * zo, (prec, k)
    print(f"TGV 128^3 10 steps: worst normwise error fp64 {worst[H.HGKS_FP64]:.2e}, fp32 {worst[H.HGKS_FP32]:.2e}")


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_uniform_flow_bitwise(precision):
    # O-P1: every face sees bitwise-identical inputs, so every face flux of a direction is
    # bitwise identical (checked on the face arrays), L == d_t L == 0 exactly, and Q never moves
    n = (16, 12, 10)
    q = inputs.uniform(n, rho=1.2, vel=(0.3, -0.7, 0.45), p=0.9)
    with _solver(n, (0, 0, 0), (1.6, 1.2, 1.0), mu=1e-3, dt_fixed=0.01, precision=precision) as s:
        s.set_state(q)
        q0 = s.get_state()
        L, dL = H.hgks_test_operator(s.ctx, 0.01, q.shape)
        assert np.all(L == 0) and np.all(dL == 0)
        for d in range(3):
            F = H.hgks_test_face_flux(s.ctx, d, n)
            assert all(np.unique(F[k]).size == 1 for k in range(10)), d
        s.step(3)
        np.testing.assert_array_equal(s.get_state(), q0)


def test_conservation_and_symmetry_gpu():
    q, dx = inputs.tgv(16)
    with _tgv_solver(16, cfl=0.4) as s:
        s.set_state(q)
        s.step(4)
        q2 = s.get_state()
    _check_conservation(q, q2, 1e-12)
    from tests.test_oracle_step import _tgv_sym_checks
    _tgv_sym_checks(q2, 1e-13)


def _check_conservation(q0, q1, rel):
    """periodic box: sum of each conservative variable is invariant (O-P2); the momenta share the
    scale sum|rho U| (TGV rhoW sums to 0 exactly)."""
    mom = math.fsum(np.sqrt((q0[1:4] ** 2).sum(0)).ravel())
    scale = [math.fsum(np.abs(q0[0]).ravel()), mom, mom, mom, math.fsum(np.abs(q0[4]).ravel())]
    for v in range(5):
        drift = abs(math.fsum(q1[v].ravel()) - math.fsum(q0[v].ravel()))
        assert drift <= rel * scale[v], (v, drift, scale[v])


def test_invalid_state_reported_with_location():
    q = inputs.uniform((8, 8, 8))
    q[4, 5, 2, 3] = -1.0  # negative energy at (i,j,k) = (3,2,5)
    with _solver((8, 8, 8), (0, 0, 0), (1, 1, 1), mu=1e-3, cfl=0.4) as s:
        with pytest.raises(H.HgksError) as e:
            s.set_state(q)
        assert e.value.code == H.HGKS_ESTATE
        assert "(3,2,5)" in str(e.value)


def test_blowup_rolls_back():
    q, dx = inputs.tgv(16)
    with _tgv_solver(16, dt_fixed=5.0) as s:  # absurd dt: the first step is invalid
        s.set_state(q)
        q0 = s.get_state()
        with pytest.raises(H.HgksError) as e:
            s.step(3)
        assert e.value.code == H.HGKS_ESTATE
        np.testing.assert_array_equal(s.get_state(), q0)
        assert s.t == 0.0


def test_t_end_clamp():
    q, dx = inputs.tgv(16)
    with _tgv_solver(16, cfl=0.4) as s:
        s.set_state(q)
        s.step(100, t_end=0.05)
        assert s.t == pytest.approx(0.05, rel=1e-14)


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_graph_replay_bitwise(precision, monkeypatch):
    """Pairs of steps replayed as CUDA graphs (default) against the plain launch path (HGKS_GRAPHS=0):
    identical bits for odd and even step counts, both buffer parities and the chunked t_end path."""
    q, dx = inputs.perturbed((20, 18, 12), seed=9, amp=0.08)

    def run(env):
        if env is None:
            monkeypatch.delenv("HGKS_GRAPHS", raising=False)
        else:
            monkeypatch.setenv("HGKS_GRAPHS", env)
        with _solver((20, 18, 12), (0.0,) * 3, (2 * math.pi,) * 3, mu=2e-3, cfl=0.4, precision=precision) as s:
            s.set_state(q)
            out = []
            for n in (2, 5, 1, 4):  # parities 0, 0 -> 1, 1 -> 0, 0
                s.step(n)
                out.append(s.get_state())
            s.step(1_000_000, t_end=s.t + 0.2)
            out.append(s.get_state())
            return out, s.t
    g, tg = run(None)
    p, tp = run("0")
    assert tg == tp
    for a, b in zip(g, p):
        assert np.array_equal(a, b)


def _gpu_wave_error(n, T=0.2):
    """3-D diagonal density wave (k = (1,1,1), U = (1,1,1), tau = 0) advected to T on the GPU; L1
    error of rho against the exact cell averages (4-point Gauss-Legendre per axis)."""
    q, h = inputs.density_wave(n, k=(1, 1, 1), vel=(1.0, 1.0, 1.0))
    steps = int(math.ceil(T / (0.1 * h[0])))
    with _solver((n, n, n), (0.0,) * 3, (2.0,) * 3, mu=0.0, dt_fixed=T / steps) as s:
        s.set_state(q)
        s.step(steps)
        got = s.get_state()[0]
    gx, gw = np.polynomial.legendre.leggauss(4)
    xc = inputs.cell_centres(n, 0.0, 2.0)
    ex = np.zeros((n, n, n))
    for a, wa in zip(gx, gw):
        for b, wb in zip(gx, gw):
            for c, wc in zip(gx, gw):
                Z, Y, X = np.meshgrid(xc + 0.5 * h[2] * c, xc + 0.5 * h[1] * b, xc + 0.5 * h[0] * a, indexing="ij")
                ex += wa * wb * wc / 8 * (1 + 0.2 * np.sin(math.pi * ((X - T) + (Y - T) + (Z - T))))
    return np.abs(got - ex).mean()


def test_fifth_order_convergence_3d_wave_gpu():
    """O-P4 on the GPU path in 3-D (every sweep, both tangential Gauss abscissae): L1 order >= 4.5."""
    errs = [_gpu_wave_error(n) for n in (16, 32, 64)]
    orders = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert min(orders) >= 4.5, (errs, orders)


def test_t_end_many_steps_chunked():
    """hgks_step with a t_end enqueues in chunks and stops at the halt: a huge nsteps costs nothing,
    and splitting the call anywhere gives the same bits (same dt sequence, same commits)."""
    import time
    q, dx = inputs.tgv(16)
    with _tgv_solver(16, cfl=0.4) as a, _tgv_solver(16, cfl=0.4) as b:
        a.set_state(q)
        b.set_state(q)
        t0 = time.perf_counter()
        a.step(1_000_000, t_end=0.5)  # ~35 steps, several chunks
        assert time.perf_counter() - t0 < 20.0
        b.step(5, t_end=0.5)
        b.step(17, t_end=0.5)
        b.step(1_000_000, t_end=0.5)
        assert a.t == pytest.approx(0.5, rel=1e-14) and b.t == a.t
        assert np.array_equal(a.get_state(), b.get_state())


def test_full_size_tgv512_sampled_parity():
    """BASELINE config 5 size on one GPU (5.4 GB per state): one CFL step at 512^3 fp64, sampled
    cells against the oracle; dt against Table 3's 512^3 value (4.462e-4)."""
    n = 512
    q, dx = inputs.tgv(n)
    with _tgv_solver(n, cfl=0.4) as s:
        s.set_state(q)
        dt = s.step(1)
        q1 = s.get_state()
    gas = O.make_gas(mu=TGV["mu"])
    dt_o = O.cfl_dt(gas, q, dx, 0.4)
    assert dt == pytest.approx(dt_o, rel=1e-13)
    assert dt_o == pytest.approx(4.462e-4, rel=1e-3)
    rng = np.random.default_rng(512)
    cells = [(0, 0, 0), (n - 1, n - 1, n - 1), (n // 2, n - 1, 1)]
    cells += [tuple(int(x) for x in rng.integers(0, n, 3)) for _ in range(9)]
    den = np.array([np.abs(q1[0]).max(), *[np.sqrt((q1[1:4] ** 2).sum(0)).max()] * 3, np.abs(q1[4]).max()])
    for c in cells:
        ref = _oracle_one_step_at(q, dx, dt_o, gas, c)
        got = q1[:, c[2], c[1], c[0]]
        assert (np.abs(got - ref) / den).max() <= 1e-11, (c, got, ref)


def _oracle_one_step_at(qfull, dx, dt, gas, cell):
    """Exact oracle value of one full S2O4 step at one cell of a periodic field, from the
    13^3 neighbourhood it depends on (stage-1 operator on 7^3, stage-2 operator at the cell)."""
    i, j, k = cell
    nz, ny, nx = qfull.shape[1:]
    ks, js, is_ = [(np.arange(-6, 7) + c) % n for c, n in ((k, nz), (j, ny), (i, nx))]
    blk = np.ascontiguousarray(qfull[:, ks][:, :, js][:, :, :, is_])
    L, dL = O.operator(gas, np.zeros((5, 7, 7, 7)), dx, dt, qg=blk)
    inner = blk[:, 3:10, 3:10, 3:10]
    qs = O.s2o4_stage1(inner, L, dL, dt)
    Ls, dLs = O.operator(gas, np.zeros((5, 1, 1, 1)), dx, dt, qg=np.ascontiguousarray(qs))
    c = (slice(None), slice(3, 4), slice(3, 4), slice(3, 4))
    return O.s2o4_final(inner[c], L[c], dL[c], dLs, dt)[:, 0, 0, 0]


@pytest.mark.parametrize("precision,tol", [(H.HGKS_FP64, 1e-11), (H.HGKS_FP32, 1e-4)])
def test_full_size_tgv256_sampled_parity(precision, tol):
    """BASELINE config 3 size, in bench.py's launch configuration: one CFL step at 256^3, 24
    sampled cells (seeded; includes domain corners and slab-boundary planes) against the oracle."""
    n = 256
    q, dx = inputs.tgv(n)
    with _tgv_solver(n, cfl=0.4, precision=precision) as s:
        s.set_state(q)
        dt = s.step(1)
        q1 = s.get_state()
    gas = O.make_gas(mu=TGV["mu"])
    dt_o = O.cfl_dt(gas, q, dx, 0.4)
    assert dt == pytest.approx(dt_o, rel=1e-13 if precision == H.HGKS_FP64 else 1e-6)
    assert dt_o == pytest.approx(8.925e-4, rel=1e-3)  # Table 3
    rng = np.random.default_rng(256)
    cells = [(0, 0, 0), (n - 1, n - 1, n - 1), (0, n - 1, 3), (n // 2, 7, n - 3)]
    cells += [tuple(int(x) for x in rng.integers(0, n, 3)) for _ in range(20)]
    den = np.array([np.abs(q1[0]).max(), *[np.sqrt((q1[1:4] ** 2).sum(0)).max()] * 3, np.abs(q1[4]).max()])
    for c in cells:
        ref = _oracle_one_step_at(q, dx, dt_o, gas, c)
        got = q1[:, c[2], c[1], c[0]]
        assert (np.abs(got - ref) / den).max() <= tol, (c, got, ref)
    # a property that holds at any size: discrete conservation (fp32: per-cell rounding of the update)
    _check_conservation(q, q1, 1e-12 if precision == H.HGKS_FP64 else 1e-6)
