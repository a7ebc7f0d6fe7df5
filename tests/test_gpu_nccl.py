"""The NCCL transport of the slab decomposition (hgks.cu coll_halo / coll_allreduce /
ncclCommInitRank) on >= 2 GPUs, one process per GPU: the gathered state after 3 CFL
steps must equal the single-domain run BITWISE (decomposition invariance, SURVEY O-P15), as the
loopback transport already shows on one GPU.  Skips when fewer than 2 devices are visible; the
one-GPU dry run of the same multi-rank bench path is test_bench_loopback_two_ranks."""
import json
import math
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2207_01173_b200 import hgks as H
from paper_2207_01173_b200 import inputs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_nccl_two_ranks_bitwise(tmp_path, precision):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (NCCL refuses two ranks on one device; see test_gpu_decomposition)")
    out = tmp_path / "nccl.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "nccl_worker.py"),
           "--out", str(out), "--precision", str(precision)]
    subprocess.run(cmd, check=True, timeout=600, cwd=ROOT)
    got = np.load(out)
    grid = (20, 18, 23)
    q, _ = inputs.perturbed(grid, seed=5, amp=0.08)
    with H.Solver(grid, (0.0,) * 3, (2 * math.pi,) * 3, mu=2e-3, cfl=0.4, precision=precision, device=0) as s:
        s.set_state(q)
        s.step(3)
        ref = s.get_state()
        t_ref = s.t
        diag = s.diagnostics()
    assert np.all(got["t"] == t_ref), (got["t"], t_ref)
    assert np.array_equal(got["state"], ref), np.abs(got["state"] - ref).max()
    assert np.array_equal(got["state_leg2"], ref)  # a second context with a fresh unique id
    d_ref = np.array([diag[k] for k in H.DIAG_NAMES])
    assert np.allclose(got["diag"], d_ref, rtol=1e-12, atol=1e-14)


def test_bench_loopback_two_ranks():
    """`bench.py --gpus 2 --transport loopback` runs the whole N-rank bench path on one GPU and
    prints one line with n_gpus = 2."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--transport", "loopback", "--n", "64",
           "--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e"]
    r = subprocess.run(cmd, check=True, timeout=600, cwd=ROOT, capture_output=True, text=True)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["transport"] == "loopback"
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["fp32"]["value"] > 0


@pytest.mark.parametrize("precision", [H.HGKS_FP64, H.HGKS_FP32])
def test_nccl_one_member_communicator_bitwise(precision):
    """The NCCL transport on ONE GPU: a context given an NCCL unique id with nranks = 1 creates a
    one-member communicator (ncclCommInitRank + ncclCommSplit), runs each stage's periodic z wrap
    as a grouped NCCL self send/recv on the communication stream and the CFL word / diagnostics as
    NCCL allreduces -- the calls of coll_halo / coll_allreduce that P > 1 uses.  It must reproduce
    the device-copy path bitwise (3 CFL steps, state, times and diagnostics), for two contexts in a
    row (each with a fresh id)."""
    grid = (20, 18, 23)
    q, _ = inputs.perturbed(grid, seed=5, amp=0.08)
    kw = dict(mu=2e-3, cfl=0.4, precision=precision, device=0)
    with H.Solver(grid, (0.0,) * 3, (2 * math.pi,) * 3, **kw) as s:
        s.set_state(q)
        s.step(3)
        ref, t_ref, d_ref = s.get_state(), s.t, s.diagnostics()
    for _ in range(2):
        with H.Solver(grid, (0.0,) * 3, (2 * math.pi,) * 3, nccl_id=H.hgks_get_nccl_id(), **kw) as s:
            s.set_state(q)
            s.step(3)
            got, t_got, d_got = s.get_state(), s.t, s.diagnostics()
        assert t_got == t_ref
        assert np.array_equal(got, ref), np.abs(got - ref).max()
        for k in H.DIAG_NAMES:
            assert d_got[k] == d_ref[k], (k, d_got[k], d_ref[k])


def test_nccl_worker_one_rank_torchrun(tmp_path):
    """tests/nccl_worker.py (the multi-rank NCCL test's worker: torch.distributed bootstrap, fresh id
    per context broadcast from rank 0, gather) under torch.distributed.run with ONE rank, which
    takes the one-member-communicator path: bitwise equal to the plain single-domain run."""
    out = tmp_path / "nccl1.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "nccl_worker.py"),
           "--out", str(out), "--precision", str(H.HGKS_FP64), "--self-comm"]
    subprocess.run(cmd, check=True, timeout=600, cwd=ROOT)
    got = np.load(out)
    grid = (20, 18, 23)
    q, _ = inputs.perturbed(grid, seed=5, amp=0.08)
    with H.Solver(grid, (0.0,) * 3, (2 * math.pi,) * 3, mu=2e-3, cfl=0.4, device=0) as s:
        s.set_state(q)
        s.step(3)
        ref = s.get_state()
    assert np.array_equal(got["state"], ref) and np.array_equal(got["state_leg2"], ref)


def test_bench_nccl_self():
    """`bench.py --transport nccl-self` (one rank, one-member NCCL communicator) prints one line."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--transport", "nccl-self", "--n", "64",
           "--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e"]
    r = subprocess.run(cmd, check=True, timeout=600, cwd=ROOT, capture_output=True, text=True)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 1 and line["config"]["transport"].startswith("nccl")
    assert line["value"] > 0 and line["fp32"]["value"] > 0
