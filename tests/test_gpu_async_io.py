"""Asynchronous host I/O of the C ABI (hgks.h: hgks_upload_state / hgks_commit_state /
hgks_download_state / hgks_io_wait): the copies run on the context's I/O stream beside the steps
(the per-rank input / output of P:554-560).  They must be exactly the synchronous set_state / get_state:
bitwise equal states, the same validity errors, and a pipelined loop (next input uploading while a step
computes, a result downloading while the next step computes) equal to the synchronous loop."""
import math

import numpy as np
import pytest

from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs

pytestmark = pytest.mark.gpu

GRID = (20, 18, 23)
KW = dict(mu=2e-3, cfl=0.4, device=0)


def _pinned(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_upload_commit_download_equal_sync(precision):
    q, _ = inputs.perturbed(GRID, seed=7, amp=0.08)
    with H.Solver(GRID, (0.0,) * 3, (2 * math.pi,) * 3, precision=precision, **KW) as s:
        s.set_state(q)
        s.step(3)
        ref = s.get_state()
    qh = _pinned(q)
    out = _pinned(np.zeros_like(q))
    with H.Solver(GRID, (0.0,) * 3, (2 * math.pi,) * 3, precision=precision, **KW) as s:
        s.upload_state(qh)
        s.commit_state()
        s.step(3)
        s.download_state(out)
        s.io_wait()
        got = out.numpy().copy()
        assert np.array_equal(got, ref), np.abs(got - ref).max()
        assert np.array_equal(s.get_state(), ref)


def test_pipelined_loop_equals_sync_loop():
    """k = 0..3: step k's input is a different seeded state each time (uploaded while step k-1 runs), its
    result downloads while step k+1 runs; every result equals set_state -> step -> get_state."""
    qs = [inputs.perturbed(GRID, seed=10 + k, amp=0.06)[0] for k in range(4)]
    refs = []
    with H.Solver(GRID, (0.0,) * 3, (2 * math.pi,) * 3, **KW) as s:
        for q in qs:
            s.set_state(q)
            s.step(1)
            refs.append(s.get_state())
    ins = [_pinned(q) for q in qs]
    outs = [_pinned(np.zeros_like(q)) for q in qs]
    with H.Solver(GRID, (0.0,) * 3, (2 * math.pi,) * 3, **KW) as s:
        s.upload_state(ins[0])
        s.commit_state()
        for k in range(4):
            if k + 1 < 4:
                s.upload_state(ins[k + 1])
            s.step(1)
            s.download_state(outs[k])
            if k + 1 < 4:
                s.commit_state()
        s.io_wait()
    for k in range(4):
        assert np.array_equal(outs[k].numpy(), refs[k]), k


def test_async_io_errors():
    q, _ = inputs.perturbed(GRID, seed=3, amp=0.05)
    with H.Solver(GRID, (0.0,) * 3, (2 * math.pi,) * 3, **KW) as s:
        with pytest.raises(H.HgksError) as e:
            s.commit_state()  # no pending upload
        assert e.value.code == H.HGKS_EINVAL
        with pytest.raises(H.HgksError) as e:
            s.download_state(_pinned(np.zeros_like(q)))  # no state yet
        assert e.value.code == H.HGKS_EINVAL
        bad = q.copy()
        bad[0, 4, 5, 6] = -1.0  # rho < 0: commit must report it exactly like set_state
        s.upload_state(_pinned(bad))
        with pytest.raises(H.HgksError) as e:
            s.commit_state()
        assert e.value.code == H.HGKS_ESTATE and "(6,5,4)" in str(e.value)
        s.io_wait()


def test_async_io_loopback_two_ranks():
    """The asynchronous calls on a 2-slab decomposition (loopback group, one GPU): hgks_commit_state is
    collective (the first wave speed is allreduced), each rank uploads / downloads its own slab; the
    gathered result equals the single-domain synchronous run bitwise."""
    q, _ = inputs.perturbed(GRID, seed=21, amp=0.06)
    with H.Solver(GRID, (0.0,) * 3, (2 * math.pi,) * 3, **KW) as s:
        s.set_state(q)
        s.step(2)
        ref = s.get_state()

    def work(rank, nranks, key):
        with H.Solver(GRID, (0.0,) * 3, (2 * math.pi,) * 3, rank=rank, nranks=nranks, group_key=key, **KW) as r:
            local = np.ascontiguousarray(q[:, r.z0:r.z0 + r.nz_local])
            inp, out = _pinned(local), _pinned(np.zeros_like(local))
            r.upload_state(inp)
            r.commit_state()
            r.step(1)
            r.upload_state(inp)  # next input while nothing else is pending: re-commit the same state
            r.download_state(out)
            r.io_wait()
            mid = out.numpy().copy()
            r.set_state(mid)     # continue from the downloaded state: 1 + 1 steps
            r.step(1)
            r.download_state(out)
            r.io_wait()
            return r.z0, out.numpy().copy()

    parts = H.run_loopback_group(2, work)
    got = np.concatenate([p for _, p in sorted(parts, key=lambda t: t[0])], axis=1)
    assert np.array_equal(got, ref), np.abs(got - ref).max()
