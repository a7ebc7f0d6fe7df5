"""Probe: can two NCCL ranks share one GPU?  (torchrun --nproc-per-node 2, both on cuda:0.)
If NCCL accepts it, run a 2-rank NCCL TGV step and compare with the 1-rank result bitwise."""
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_01173_b200 import hgks as H  # noqa: E402
from paper_2207_01173_b200 import inputs  # noqa: E402

rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
obj = [H.hgks_get_nccl_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
grid = (20, 18, 24)
q, _ = inputs.perturbed(grid, seed=5, amp=0.08)
kw = dict(mu=2e-3, cfl=0.4)
try:
    s = H.Solver(grid, (0.0,) * 3, (2 * math.pi,) * 3, rank=rank, nranks=ws, nccl_id=obj[0], device=0, **kw)
except H.HgksError as e:
    print(f"rank {rank}: NCCL ranks sharing one GPU refused: {e}", flush=True)
    sys.exit(0)
s.set_state(np.ascontiguousarray(q[:, s.z0:s.z0 + s.nz_local]))
s.step(4)
got = s.get_state()
parts = [None] * ws
dist.all_gather_object(parts, (s.z0, got, s.t))
s.close()
if rank == 0:
    with H.Solver(grid, (0.0,) * 3, (2 * math.pi,) * 3, **kw) as r:
        r.set_state(q)
        r.step(4)
        ref = r.get_state()
    full = np.zeros_like(q)
    for z0, g, _ in parts:
        full[:, z0:z0 + g.shape[1]] = g
    print(f"NCCL 2 ranks on one GPU: bitwise equal to 1 rank: {np.array_equal(full, ref)}, "
          f"max diff {np.abs(full - ref).max():.3e}, t = {[p[2] for p in parts]} vs {r.t}", flush=True)
dist.destroy_process_group()
