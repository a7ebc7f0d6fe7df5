"""Multi-rank host logic on CPU (world size 2 and 3, gloo): the slab split (hgks_slab_of) and the
z-halo plan (hgks_make_halo_plan) that hgks_step hands to NCCL, exercised by exchanging real slabs
with torch.distributed send/recv exactly as the plan says, then evaluating the oracle operator on each
rank's ghosted slab.  The gathered result must equal the single-domain oracle operator bitwise
(SURVEY O-P15: decomposition invariance)."""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

N = (10, 9, 12)  # nx, ny, nz (global)
DT = 0.01
MU = 2e-3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ghosted_gpu_layout(qslab, nx, ny, nzl):
    """[5][nzl][ny][nx] -> library layout [nzl+6][5][ny+6][nx+6] with periodic x/y ghosts
    (ghost_xy_kernel semantics); z ghosts left zero for the halo exchange."""
    g = np.zeros((nzl + 6, 5, ny + 6, nx + 6))
    g[3:nzl + 3, :, 3:ny + 3, 3:nx + 3] = np.transpose(qslab, (1, 0, 2, 3))
    yi = (np.arange(-3, ny + 3)) % ny
    xi = (np.arange(-3, nx + 3)) % nx
    g[3:nzl + 3] = g[3:nzl + 3][:, :, yi + 3][:, :, :, xi + 3]
    return g


def _worker(rank, world, port, out_path):
    import torch

    from oracle import oracle as O
    from paper_2207_01173_b200 import hgks as H
    from paper_2207_01173_b200 import inputs

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz = N
    z0, nzl = H.hgks_slab_of(nz, rank, world)
    q, dx = inputs.perturbed(N, seed=11, amp=0.08)
    g = _ghosted_gpu_layout(q[:, z0:z0 + nzl], nx, ny, nzl)
    plan = H.hgks_make_halo_plan(nx, ny, nzl, rank, world)
    flat = g.reshape(-1)
    cnt = plan["count"]
    t = lambda off: torch.from_numpy(flat[off:off + cnt].copy())
    # grouped exchange as in fill_ghosts(): send top planes up / bottom planes down
    recv_dn, recv_up = torch.empty(cnt, dtype=torch.float64), torch.empty(cnt, dtype=torch.float64)
    reqs = [dist.isend(t(plan["send_up"]), plan["up"]), dist.irecv(recv_dn, plan["down"]),
            dist.isend(t(plan["send_down"]), plan["down"]), dist.irecv(recv_up, plan["up"])]
    for r in reqs:
        r.wait()
    flat[plan["recv_down"]:plan["recv_down"] + cnt] = recv_dn.numpy()
    flat[plan["recv_up"]:plan["recv_up"] + cnt] = recv_up.numpy()
    # to the oracle's ghosted layout [5][nz+6][ny+6][nx+6] and evaluate this slab's operator
    og = np.ascontiguousarray(np.transpose(g, (1, 0, 2, 3)))
    L, dL = O.operator(O.make_gas(mu=MU), np.zeros((5, nzl, ny, nx)), dx, DT, qg=og)
    parts = [None] * world
    dist.all_gather_object(parts, (z0, L, dL))
    if rank == 0:
        np.savez(out_path, *[np.concatenate([p[1], p[2]]) for p in sorted(parts, key=lambda p: p[0])])
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_halo_plan_reproduces_single_domain(world, tmp_path):
    from oracle import oracle as O
    from paper_2207_01173_b200 import inputs
    out = str(tmp_path / "parts.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    parts = [got[f"arr_{i}"] for i in range(world)]
    LdL = np.concatenate(parts, axis=1)  # along z
    q, dx = inputs.perturbed(N, seed=11, amp=0.08)
    L, dL = O.operator(O.make_gas(mu=MU), q, dx, DT)
    np.testing.assert_array_equal(LdL[:5], L)
    np.testing.assert_array_equal(LdL[5:], dL)
