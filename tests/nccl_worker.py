"""Worker of tests/test_gpu_nccl.py (launched by torch.distributed.run, one rank per GPU): runs the
NCCL slab path of libhgks (ncclCommInitRank + split halo communicator, grouped send/recv halos,
max-allreduce of the CFL word, sum-allreduce of the diagnostics) and writes the gathered state,
the times and the diagnostics to an .npz on rank 0."""
import argparse
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_01173_b200 import hgks as H  # noqa: E402
from paper_2207_01173_b200 import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--precision", type=int, default=H.HGKS_FP64)
    ap.add_argument("--self-comm", action="store_true", help="one rank: pass an id anyway (one-member communicator)")
    a = ap.parse_args()
    rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    grid = (20, 18, 23)
    q, _ = inputs.perturbed(grid, seed=5, amp=0.08)
    results = {}
    for leg in range(2):  # two contexts in a row: each needs its own unique id (bootstrap serves one init)
        obj = [H.hgks_get_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        if ws == 1 and not a.self_comm:
            obj = [None]
        s = H.Solver(grid, (0.0,) * 3, (2 * math.pi,) * 3, mu=2e-3, cfl=0.4, precision=a.precision, rank=rank,
                     nranks=ws, device=local, nccl_id=obj[0])
        s.set_state(np.ascontiguousarray(q[:, s.z0:s.z0 + s.nz_local]))
        s.step(a.steps)
        diag = s.diagnostics()
        parts = [None] * ws
        dist.all_gather_object(parts, (s.z0, s.get_state(), s.t))
        s.close()
        results[leg] = (parts, diag)
    if rank == 0:
        out = np.zeros_like(q)
        ts = []
        for z0, st, t in results[0][0]:
            out[:, z0:z0 + st.shape[1]] = st
            ts.append(t)
        out1 = np.zeros_like(q)
        for z0, st, _ in results[1][0]:
            out1[:, z0:z0 + st.shape[1]] = st
        np.savez(a.out, state=out, state_leg2=out1, t=np.array(ts),
                 diag=np.array([results[0][1][k] for k in H.DIAG_NAMES]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
