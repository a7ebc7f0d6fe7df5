"""Slab decomposition on ONE GPU through the in-process loopback group (hgks_params.group_key):
nranks contexts on host threads, same kernels, slab split (hgks_slab_of) and halo plan
(hgks_make_halo_plan) as the NCCL path, halos moved by device copies on the communication stream,
reductions in a fixed rank order.

SURVEY O-P15 (decomposition invariance): the step is a per-cell function of a +-3 neighbourhood and
the CFL reduction is an exact max, so the gathered state after n steps must equal the single-domain
run BITWISE for any slab split, including uneven ones.  Sums (diagnostics, plane statistics, the
bulk-force controller) change their rounding order with the split, so those compare to round-off.
"""
import math

import numpy as np
import pytest

from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs

pytestmark = pytest.mark.gpu
TGV = inputs.tgv_params()


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device (no CPU fallback exists)"
    H.lib()


def _run(nranks, grid, q_global, steps, kw, per_rank=None):
    """Run `steps` steps on nranks loopback ranks; returns (gathered state, [t], [extra])."""
    def work(rank, n, key):
        s = H.Solver(grid, kw["lo"], kw["hi"], rank=rank, nranks=n, group_key=key if n > 1 else 0,
                     **{k: v for k, v in kw.items() if k not in ("lo", "hi")})
        try:
            s.set_state(np.ascontiguousarray(q_global[:, s.z0:s.z0 + s.nz_local]))
            s.step(steps)
            extra = per_rank(s) if per_rank else None
            return s.z0, s.get_state(), s.t, extra
        finally:
            s.close()
    res = H.run_loopback_group(nranks, work) if nranks > 1 else [work(0, 1, 0)]
    out = np.zeros_like(q_global)
    for z0, q, _, _ in res:
        out[:, z0:z0 + q.shape[1]] = q
    return out, [r[2] for r in res], [r[3] for r in res]


def _tgv_kw(precision):
    return dict(lo=(0.0,) * 3, hi=(2 * math.pi,) * 3, mu=2e-3, cfl=0.4, precision=precision)


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_slab_split_bitwise_ragged(nranks, precision):
    grid = (20, 18, 23)  # ragged in every axis; 23 planes split unevenly (e.g. 5,5,5,4,4)
    q, _ = inputs.perturbed(grid, seed=5, amp=0.08)
    kw = _tgv_kw(precision)
    ref, t1, _ = _run(1, grid, q, 4, kw)
    got, tn, _ = _run(nranks, grid, q, 4, kw)
    assert all(t == t1[0] for t in tn), (t1, tn)  # global CFL dt: identical on every rank
    assert np.array_equal(got, ref), np.abs(got - ref).max()


def test_tgv128_four_slabs_bitwise():
    n = 128
    q, _ = inputs.tgv(n)
    kw = dict(lo=(-math.pi,) * 3, hi=(math.pi,) * 3, mu=TGV["mu"], cfl=0.4)
    ref, t1, _ = _run(1, (n, n, n), q, 2, kw)
    got, tn, _ = _run(4, (n, n, n), q, 2, kw)
    assert tn == [t1[0]] * 4
    assert np.array_equal(got, ref)


def _channel_kw(precision):
    c = inputs.channel_params()
    return dict(lo=c["lo"], hi=c["hi"], mu=c["mu_w"], mu_law=H.HGKS_MU_POWER, T_ref=c["T_w"], omega=c["omega"],
                prandtl=c["prandtl"], T_wall=c["T_w"], bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                stretch=(H.HGKS_UNIFORM, H.HGKS_TANH, H.HGKS_UNIFORM), stretch_b=(0.0, c["b_g"], 0.0), cfl=0.4,
                precision=precision)


def test_channel_walls_stretched_split_bitwise():
    grid = (16, 24, 15)
    q = inputs.channel(grid)[0]
    kw = _channel_kw(H.HGKS_FP64)
    ref, _, _ = _run(1, grid, q, 3, kw)
    got, _, _ = _run(3, grid, q, 3, kw)
    assert np.array_equal(got, ref)


def test_channel_bulk_forcing_split_roundoff():
    """O-27 controller: the bulk sums are reduced per rank then summed over the group, so the force
    (and through it the state) agrees with the single-domain run to round-off, not bitwise."""
    grid = (16, 24, 16)
    q = inputs.channel(grid)[0]
    kw = dict(_channel_kw(H.HGKS_FP64), force_mode=H.HGKS_FORCE_BULK, force=0.0, force_target=1.0)
    forcing = lambda s: H.hgks_get_forcing(s.ctx)  # noqa: E731
    ref, _, f1 = _run(1, grid, q, 4, kw, forcing)
    got, _, fn = _run(2, grid, q, 4, kw, forcing)
    for f in fn:
        # m, rho_b: sums of ~4e3 terms, round-off only; f = (m_b - m)/dt / rho_b amplifies the
        # O(1e-16) rounding of m by 1/dt (dt ~ 1e-3 here): absolute 1e-12 on f ~ 1e-3
        assert np.allclose(f[1:], f1[0][1:], rtol=1e-14, atol=0), (f, f1[0])
        assert abs(f[0] - f1[0][0]) <= 1e-12, (f, f1[0])
    for v in range(5):
        den = np.abs(ref[v]).max() if v in (0, 4) else np.sqrt((ref[1:4] ** 2).sum(0)).max()
        assert np.abs(got[v] - ref[v]).max() / den <= 1e-13


def test_diagnostics_and_plane_stats_global():
    grid = (16, 24, 12)
    q = inputs.channel(grid)[0]
    kw = _channel_kw(H.HGKS_FP64)
    both = lambda s: (H.hgks_diagnostics(s.ctx), s.plane_stats())  # noqa: E731
    _, _, e1 = _run(1, grid, q, 1, kw, both)
    _, _, en = _run(4, grid, q, 1, kw, both)
    d1, p1 = e1[0]
    for dn, pn in en:  # every rank receives the global values
        assert np.allclose(dn, d1, rtol=1e-13, atol=1e-14 * np.abs(d1).max())
        assert np.allclose(pn, p1, rtol=1e-12, atol=1e-13 * np.abs(p1).max())


def test_invalid_state_on_one_rank_reported_everywhere():
    grid = (12, 12, 12)
    q, _ = inputs.perturbed(grid, seed=2, amp=0.05)
    q[0, 10, 3, 4] = -1.0  # rho < 0 in rank 1's slab (planes 6..11 of 2 ranks)

    def work(rank, n, key):
        s = H.Solver(grid, (0.0,) * 3, (2 * math.pi,) * 3, mu=1e-3, cfl=0.4, rank=rank, nranks=n, group_key=key)
        try:
            with pytest.raises(H.HgksError) as ei:
                s.set_state(np.ascontiguousarray(q[:, s.z0:s.z0 + s.nz_local]))
            return ei.value.code, str(ei.value)
        finally:
            s.close()
    res = H.run_loopback_group(2, work)
    assert [r[0] for r in res] == [H.HGKS_ESTATE] * 2
    assert "(4,3,10)" in res[1][1] and "another rank" in res[0][1]


def test_group_key_validation():
    with pytest.raises(H.HgksError) as ei:
        H.Solver((8, 8, 8), (0,) * 3, (1,) * 3, cfl=0.4, nranks=2, rank=0)
    assert ei.value.code == H.HGKS_EINVAL
