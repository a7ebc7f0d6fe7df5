"""Per-call host timing of the asynchronous-I/O loop (bench.py e2e) at TGV n^3: where does the time go?
usage: python tools/async_io_timing.py [n] [steps]"""
import math
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_01173_b200 import hgks as H  # noqa: E402
from paper_2207_01173_b200 import inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
q, _ = inputs.tgv(n)
qh = torch.from_numpy(q).pin_memory()
qo = torch.empty_like(qh).pin_memory()
with H.Solver((n,) * 3, (-math.pi,) * 3, (math.pi,) * 3, mu=inputs.tgv_params()["mu"], cfl=0.4) as s:
    s.set_state(qh.numpy())
    s.step(3)
    s.upload_state(qh); s.commit_state(); s.download_state(qo); s.io_wait()
    t = time.perf_counter()
    s.step(steps)
    print(f"plain step: {(time.perf_counter() - t) / steps * 1e3:.2f} ms")
    t = time.perf_counter(); s.upload_state(qh); s.io_wait(); print(f"upload alone: {(time.perf_counter() - t) * 1e3:.2f} ms")
    t = time.perf_counter(); s.commit_state(); print(f"commit alone: {(time.perf_counter() - t) * 1e3:.2f} ms")
    t = time.perf_counter(); s.download_state(qo); s.io_wait(); print(f"download alone: {(time.perf_counter() - t) * 1e3:.2f} ms")
    T = {"upload": 0.0, "step": 0.0, "download": 0.0, "commit": 0.0}
    t0 = time.perf_counter()
    s.upload_state(qh); s.commit_state()
    tp = time.perf_counter() - t0
    for k in range(steps):
        a = time.perf_counter()
        if k + 1 < steps:
            s.upload_state(qh)
        b = time.perf_counter(); s.step(1); c = time.perf_counter()
        s.download_state(qo); d = time.perf_counter()
        if k + 1 < steps:
            s.commit_state()
        e = time.perf_counter()
        T["upload"] += b - a; T["step"] += c - b; T["download"] += d - c; T["commit"] += e - d
    f = time.perf_counter(); s.io_wait(); g = time.perf_counter()
    tot = g - t0
    print(f"loop: {tot / steps * 1e3:.2f} ms/step (prologue {tp*1e3:.1f} ms, final io_wait {(g-f)*1e3:.1f} ms); per step " +
          ", ".join(f"{k} {v / steps * 1e3:.2f}" for k, v in T.items()))
    # does an enqueued upload progress while the host waits / while a step runs?
    s.io_wait()
    t = time.perf_counter(); s.upload_state(qh); time.sleep(0.03); a = time.perf_counter(); s.io_wait()
    print(f"upload + 30 ms host sleep: io_wait took {(time.perf_counter() - a) * 1e3:.2f} ms")
    s.commit_state()
    t = time.perf_counter(); s.upload_state(qh); s.step(1); a = time.perf_counter(); s.io_wait()
    print(f"upload + step: step {(a - t) * 1e3:.2f} ms, io_wait after it {(time.perf_counter() - a) * 1e3:.2f} ms")
    s.commit_state()
    t = time.perf_counter(); s.download_state(qo); s.step(1); a = time.perf_counter(); s.io_wait()
    print(f"download + step: step {(a - t) * 1e3:.2f} ms, io_wait after it {(time.perf_counter() - a) * 1e3:.2f} ms")
