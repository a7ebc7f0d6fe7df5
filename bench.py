#!/usr/bin/env python
"""bench.py — HGKS S2O4 step throughput on B200 (BASELINE.json metric: cell-updates/s, TGV 256^3).

One "step" = one full two-stage S2O4 step (A0..A8 of SURVEY.md §8(a)) over the whole grid.

Launch modes (one JSON line from rank 0 in every mode):
  python bench.py                          1 GPU (N = 1)
  torchrun --nproc-per-node N bench.py --gpus N
                                           N ranks, one per GPU, NCCL z-slab halos (the driver's launch)
  python bench.py --gpus N                 same: re-executes itself under torch.distributed.run when
                                           WORLD_SIZE is unset (needs N visible GPUs)
  python bench.py --gpus N --transport loopback
                                           N slab ranks in ONE process on host threads, sharing the
                                           visible GPUs round-robin (the in-process loopback group of
                                           hgks.h: same kernels, slab split, halo plan and collectives'
                                           placement as NCCL) -- a dry run of the N-rank path on 1 GPU
  python bench.py --transport nccl-self    1 rank through a one-member NCCL communicator (halo by NCCL
                                           self send/recv, NCCL allreduce): the NCCL calls on 1 GPU
  python bench.py --impl reference         the plain CPU oracle on the host cores (reference arm)

Prints ONE JSON line on rank 0 (DESIGN.md §8 "Measurement").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/s"
N_SM = 148
# derived nominal ALU peaks (per SM per clock): 64 FP64 FMA, 128 FP32 FMA
FP64_FMA_PER_CLK, FP32_FMA_PER_CLK = 64, 128


def _json(path):
    try:
        with open(os.path.join(ROOT, path)) as f:
            return json.load(f)
    except Exception:
        return None


def _peaks():
    return _json("MEASURED_PEAKS.json") or {}


def alu_peak(kind: str, sm_max: float):
    """(TFLOP/s, source) of the FP64 (kind 'dfma') or FP32 ('ffma') FMA pipe: the committed
    microbenchmark measurement (profiles/alu_peaks.json, tools/microbench/alu_peaks.cu) when
    present, else derived from unit counts x clocks.max.sm."""
    per_clk = FP64_FMA_PER_CLK if kind == "dfma" else FP32_FMA_PER_CLK
    derived = N_SM * per_clk * 2 * sm_max * 1e6 / 1e12
    m = _json(os.path.join("profiles", "alu_peaks.json"))
    if m and m.get(kind + "_tflops"):
        return float(m[kind + "_tflops"]), (f"of measured: {kind.upper()} microbenchmark {m[kind + '_tflops']:.2f} TF "
                                            f"(profiles/alu_peaks.json; derived nominal {derived:.2f})")
    return derived, f"of derived nominal: {N_SM} SMs x {per_clk} FMA/clk x 2 x {sm_max:.0f} MHz"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------------------------
# CPU baseline: the oracle as it stands (test infrastructure; only this leg and --impl reference
# execute it)
# ---------------------------------------------------------------------------------------------
def _tgv_block(n: int, planes: int):
    from paper_2207_01173_b200 import inputs
    zidx = np.arange(-3, planes + 3) % n
    blk_z = np.concatenate([inputs.tgv(n, z_begin=int(z), nz_local=1)[0] for z in zidx], axis=1)
    w = np.arange(-3, n + 3) % n
    return np.ascontiguousarray(blk_z[:, :, w][:, :, :, w])


def cpu_operator_sample(n: int, planes: int, mu: float, threads: int = 0, stage_count: int = 2):
    """Oracle operator L, d_t L on `planes` z-planes of the TGV n^3 field (true neighbour ghosts),
    once per stage = the flux work of one S2O4 step on n*n*planes cells.  Returns
    (cell-updates/s, cores used, seconds, sample description)."""
    from oracle import oracle as O
    blk = _tgv_block(n, planes)
    gas = O.make_gas(mu=mu)
    dummy = np.zeros((5, planes, n, n))
    O.set_num_threads(threads)
    try:
        cores = O.num_threads()
        t0 = time.perf_counter()
        for _ in range(stage_count):
            O.operator(gas, dummy, (2 * math.pi / n,) * 3, 1e-3, qg=blk)
        sec = time.perf_counter() - t0
    finally:
        O.set_num_threads(0)
    return n * n * planes / sec, cores, sec, f"oracle operator on {n}x{n}x{planes} z-planes of TGV {n}^3, x{stage_count} stages"


def cpu_run_c1(threads: int = 0, steps: int = 10):
    """BASELINE config 1 in full: TGV 32^3, `steps` complete CFL S2O4 steps of the oracle."""
    from oracle import oracle as O
    from paper_2207_01173_b200 import inputs
    n = 32
    q, dx = inputs.tgv(n)
    gas = O.make_gas(mu=inputs.tgv_params()["mu"])
    O.set_num_threads(threads)
    try:
        cores = O.num_threads()
        t0 = time.perf_counter()
        O.run(gas, q, dx, steps)
        sec = time.perf_counter() - t0
    finally:
        O.set_num_threads(0)
    return n ** 3 * steps / sec, cores, sec


def cpu_baseline_block(n: int, planes: int, mu: float):
    v, cores, sec, sample = cpu_operator_sample(n, planes, mu)
    v1, _, sec1, _ = cpu_operator_sample(n, 1, mu, threads=1)
    c1, c1_cores, c1_sec = cpu_run_c1()
    c1s, _, c1s_sec = cpu_run_c1(threads=1, steps=2)
    return {"value": v, "unit": "cell-updates/s", "cores": cores, "kind": "oracle", "sample": sample,
            "seconds": sec,
            "single_thread": {"value": v1, "cores": 1, "sample": f"oracle operator on {n}x{n}x1 z-plane, x2 stages",
                              "seconds": sec1},
            "c1_tgv32_10steps": {"value": c1, "cores": c1_cores, "seconds": c1_sec,
                                 "single_thread_value": c1s, "single_thread_sample": "2 steps", "single_thread_seconds": c1s_sec}}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    n = args.n
    from paper_2207_01173_b200 import inputs
    prm = inputs.tgv_params()
    planes = 1
    times, cores, sample = [], None, ""
    for i in range(args.warmup + args.steps):
        _, cores, sec, sample = cpu_operator_sample(n, planes, prm["mu"])
        if i >= args.warmup:
            times.append(sec)
    ms = 1000 * float(np.mean(times))
    value = n * n * planes / (ms / 1000)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"tgv{n}", "grid": [n, n, n], "precision": "fp64", "mode": "cfl"},
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
                             "sample": sample + " per step"},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# rank environments: NCCL (one process per GPU) or the in-process loopback group (host threads)
# ---------------------------------------------------------------------------------------------
class NcclEnv:
    transport = "nccl"

    def __init__(self, dist, ws, rank, local, self_comm=False):
        import torch
        self.dist, self.ws, self.rank, self.device = dist, ws, rank, local
        self.self_comm = self_comm  # one rank, NCCL transport anyway (--transport nccl-self)
        self.stream = torch.cuda.Stream(device=local)

    def barrier(self):
        import torch
        if self.ws > 1:
            self.dist.barrier()
        torch.cuda.synchronize(self.device)

    def reduce(self, x: float, op: str) -> float:
        if self.ws == 1:
            return x
        import torch
        t = torch.tensor([x], device=f"cuda:{self.device}", dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def comm_kwargs(self):
        """A FRESH NCCL unique id for every context (NCCL's bootstrap root serves one init)."""
        from paper_2207_01173_b200 import hgks as H
        if self.ws == 1:
            return {"nccl_id": H.hgks_get_nccl_id()} if self.self_comm else {}
        obj = [H.hgks_get_nccl_id() if self.rank == 0 else None]
        self.dist.broadcast_object_list(obj, src=0)
        return {"nccl_id": obj[0]}


class LoopbackShared:
    def __init__(self, ws):
        self.ws = ws
        self.bar = threading.Barrier(ws)
        self.vals = [0.0] * ws
        self.keys = iter(range(os.getpid() * 1000 + 1, os.getpid() * 1000 + 1000))
        self.key = None


class LoopbackEnv:
    transport = "loopback"

    def __init__(self, shared: LoopbackShared, rank: int, ndev: int):
        import torch
        self.sh, self.ws, self.rank = shared, shared.ws, rank
        self.device = rank % ndev
        torch.cuda.set_device(self.device)
        self.stream = torch.cuda.Stream(device=self.device)

    def barrier(self):
        import torch
        self.sh.bar.wait()
        torch.cuda.synchronize(self.device)
        self.sh.bar.wait()

    def reduce(self, x: float, op: str) -> float:
        self.sh.vals[self.rank] = x
        self.sh.bar.wait()
        v = max(self.sh.vals) if op == "max" else sum(self.sh.vals)
        self.sh.bar.wait()
        return v

    def comm_kwargs(self):
        if self.rank == 0:
            self.sh.key = next(self.sh.keys)
        self.sh.bar.wait()
        key = self.sh.key
        self.sh.bar.wait()
        return {"group_key": key}


# ---------------------------------------------------------------------------------------------
# one rank's measurement (fp64 and fp32 legs)
# ---------------------------------------------------------------------------------------------
def measure_rank(args, env) -> dict | None:
    import torch

    from paper_2207_01173_b200 import hgks as H
    from paper_2207_01173_b200 import inputs

    ws, rank = env.ws, env.rank
    n = args.n
    nz = (n // 8) * ws if args.weak else n
    grid = (n, n, nz)
    prm = inputs.tgv_params()
    channel = args.workload == "channel"
    if channel:
        grid = tuple(int(x) for x in args.channel_grid.split(","))
        chp = inputs.channel_params()
    stream = env.stream
    lo, hi = (-math.pi,) * 3, (math.pi,) * 3  # weak mode: same box, nz = n/8 * N planes (anisotropic dz)

    def make_solver(precision):
        kw = dict(cfl=0.4, precision=precision, rank=rank, nranks=ws, device=env.device,
                  stream=stream.cuda_stream, **env.comm_kwargs())
        if channel:  # config 4: walls in y, tanh mesh, power-law mu, Pr = 0.7
            return H.Solver(grid, chp["lo"], chp["hi"], mu=chp["mu_w"], mu_law=H.HGKS_MU_POWER, T_ref=chp["T_w"],
                            omega=chp["omega"], prandtl=chp["prandtl"], T_wall=chp["T_w"],
                            bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                            stretch=(H.HGKS_UNIFORM, H.HGKS_TANH, H.HGKS_UNIFORM), stretch_b=(0.0, chp["b_g"], 0.0),
                            # constant bulk momentum rho_b U_b = 1 (units of the channel, O-27)
                            force_mode=H.HGKS_FORCE_BULK, force=0.0, force_target=1.0, **kw)
        return H.Solver(grid, lo, hi, mu=prm["mu"], **kw)

    def local_field(s):
        if channel:
            return inputs.channel(grid, z_begin=s.z0, nz_local=s.nz_local)[0]
        return inputs.tgv(grid, z_begin=s.z0, nz_local=s.nz_local)[0]

    results = {}
    for prec_name, prec in (("fp64", H.HGKS_FP64), ("fp32", H.HGKS_FP32)):
        if (prec_name == "fp32" and args.no_fp32) or (prec_name == "fp64" and args.only_fp32):
            continue
        torch.cuda.synchronize(env.device)
        free0 = torch.cuda.mem_get_info(env.device)[0]
        s = make_solver(prec)
        torch.cuda.synchronize(env.device)
        # device memory the library allocated for this context (Table 8's "memory cost")
        mem_bytes = free0 - torch.cuda.mem_get_info(env.device)[0]
        if ws > 1:  # evidence of the N-rank launch for the driver's log (stderr; stdout is the JSON line)
            print(f"[bench] {prec_name}: rank {rank}/{ws} on cuda:{env.device}, transport {env.transport}, "
                  f"z-slab [{s.z0}, {s.z0 + s.nz_local}) of {grid[2]}", file=sys.stderr, flush=True)
        q = local_field(s)
        with torch.cuda.device(env.device):
            qd = torch.from_numpy(q).cuda()
        s.set_state(qd)
        s.step(args.warmup)
        env.barrier()
        H.hgks_profile_enable(s.ctx, True)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(env.device) as clk:
            env.barrier()
            ev0.record(stream)
            s.step(args.steps)
            ev1.record(stream)
            env.barrier()
        ms_local = ev0.elapsed_time(ev1)
        ms_k, launches, total_launches = H.hgks_profile_read(s.ctx)
        H.hgks_profile_enable(s.ctx, False)
        ms = env.reduce(ms_local, "max")
        total_launches = int(env.reduce(float(total_launches), "sum"))
        cells = grid[0] * grid[1] * grid[2]
        rate = cells * args.steps / (ms / 1000.0)
        res = dict(ms_per_step=ms / args.steps, value=rate, clocks=clk.summary(), ms_k=ms_k, launches=launches,
                   total_launches=total_launches, t=s.t, mem_bytes=int(env.reduce(float(mem_bytes), "sum")))
        # NEXT-1/2 device reductions outside the timed step (synchronous calls, events on the stream)
        aux = {}
        for name, fn in (("diagnostics", lambda: H.hgks_diagnostics(s.ctx)),
                         ("plane_stats", lambda: H.hgks_plane_stats(s.ctx, grid[1]))):
            fn()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(3):
                fn()
            a1.record(stream)
            torch.cuda.synchronize(env.device)
            aux[name + "_ms"] = a0.elapsed_time(a1) / 3
        # per-step diagnostic history (fused into the stage-1 update): its cost per step is the growth of the
        # update-class event time (the fused diagnostics + the two reduction kernels), 6 steps each way
        def update_ms(k):
            H.hgks_profile_enable(s.ctx, True)
            s.step(k)
            ms_k2, _, _ = H.hgks_profile_read(s.ctx)
            H.hgks_profile_enable(s.ctx, False)
            return env.reduce(ms_k2["update"], "max") / k
        t_off = update_ms(6)
        H.hgks_history_enable(s.ctx, 8)
        t_on = update_ms(6)
        hist = H.hgks_history_read(s.ctx, 8)
        H.hgks_history_enable(s.ctx, 0)
        aux["history_ms_per_step"] = t_on - t_off
        aux["history_rows_read"] = int(hist.shape[0])
        res["aux"] = aux
        # e2e through the public API with host buffers (pinned): every step's input is copied host -> device
        # and its result device -> host.  Headline `e2e`: the asynchronous I/O calls (hgks_upload_state /
        # commit / download / io_wait), which run the copies on the copy engines beside the steps (the
        # next input uploads while the current step computes; a result downloads while the next step
        # computes).  `e2e_sync`: the synchronous set_state -> step -> get_state loop.
        if not args.no_e2e:
            qh = torch.from_numpy(q).pin_memory()
            qo = torch.empty_like(qh).pin_memory()
            e_steps = max(2, args.steps)
            # one untimed pass of each call first: the I/O stream and its two staging buffers are allocated
            # on first use (set-up, not per-step cost)
            s.upload_state(qh)
            s.commit_state()
            s.download_state(qo)
            s.io_wait()
            for mode in ("async", "sync"):
                env.barrier()
                t0 = time.perf_counter()
                e_ev0, e_ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e_ev0.record(stream)
                if mode == "async":
                    s.upload_state(qh)
                    s.commit_state()
                    for k in range(e_steps):
                        if k + 1 < e_steps:
                            s.upload_state(qh)  # the next step's input, while this step computes
                        s.step(1)
                        s.download_state(qo)  # this step's result, while the next step computes
                        if k + 1 < e_steps:
                            s.commit_state()
                    s.io_wait()
                else:
                    for _ in range(e_steps):
                        s.set_state(qh.numpy())
                        s.step(1)
                        s.get_state(qo.numpy())
                e_ev1.record(stream)
                torch.cuda.synchronize(env.device)
                env.barrier()
                e_ms = env.reduce(e_ev0.elapsed_time(e_ev1), "max")
                rec = {"value": cells * e_steps / (e_ms / 1000.0), "unit": "cell-updates/s",
                       "h2d_bytes_per_step": int(env.reduce(float(q.nbytes), "sum")),
                       "d2h_bytes_per_step": int(env.reduce(float(q.nbytes), "sum")),
                       "steps": e_steps, "wall_s": time.perf_counter() - t0}
                if mode == "async":
                    rec["api"] = "hgks_upload_state / commit_state / step / download_state / io_wait (copies overlap steps)"
                    res["e2e"] = rec
                else:
                    rec["api"] = "hgks_set_state / step / get_state (synchronous)"
                    res["e2e_sync"] = rec
        s.close()
        del qd
        torch.cuda.empty_cache()
        results[prec_name] = res
    if rank != 0 or args.only_fp32:
        return None
    return {"results": results, "grid": grid, "channel": channel, "prm": prm}


def flux_roofline(r, grid, ws, steps, prec: str, sm_max: float):
    """roofline of the dominant kernel (the fused flux sweeps): executed FP64/FP32 flops per launch
    (ncu SASS counts per face, profiles/flux_flops.json) / the live CUDA-event launch time."""
    flux_ms = sum(r["ms_k"][k] for k in ("flux_x", "flux_y", "flux_z"))
    flux_launches = sum(r["launches"][k] for k in ("flux_x", "flux_y", "flux_z"))
    kind = "dfma" if prec == "fp64" else "ffma"
    peak, src = alu_peak(kind, sm_max)
    roof = {"bound": "alu", "kernel": f"flux_kernel<{'double' if prec == 'fp64' else 'float'},DIR,STAGE> (x,y,z faces, both stages)",
            "peak": peak, "unit": "TFLOP/s", "peak_source": src,
            "flux_share_of_step": flux_ms / (r["ms_per_step"] * steps) if r["ms_per_step"] else None,
            "avg_launch_ms": flux_ms / flux_launches if flux_launches else None, "traffic": None}
    ftab = _json(os.path.join("profiles", "flux_flops.json"))
    key1, key2 = f"{prec}_flop_per_face_stage1", f"{prec}_flop_per_face_stage2"
    if ftab and key1 in ftab:
        gx, gy, gzl = grid[0], grid[1], grid[2] // ws
        faces = 3 * gx * gy * gzl + gy * gzl + gx * gzl + gx * gy  # x, y, z faces of one rank's slab
        flops_step = faces * (ftab[key1] + ftab[key2])
        achieved = flops_step * steps / (flux_ms / 1000.0) / 1e12
        roof.update(achieved=achieved, frac=achieved / peak,
                    flop_count="executed FP%s flops of the flux kernels (SASS: 2 x FMA + MUL + ADD, ncu), %.0f + %.0f per face "
                               "(stages 1 + 2); the method's own algebra costs more (DESIGN.md §8)" % (prec[2:], ftab[key1], ftab[key2]),
                    flop_source=ftab.get("source"), traffic=ftab.get(f"{prec}_dram_bytes_per_launch_stage1"),
                    traffic_note="ncu dram__bytes_read+write per stage-1 flux launch (same counters file)")
    return roof


def report(args, out, ws, transport):
    results, grid, channel, prm = out["results"], out["grid"], out["channel"], out["prm"]
    n = args.n
    r64 = results["fp64"]
    peaks = _peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    hbm = float(peaks.get("hbm_gbs", 6548.5))
    alg_bytes = 240.0  # fp64 bytes per cell-update
    workload = ("channel_" + "x".join(map(str, grid))) if channel else (f"tgv{n}" + ("_weak" if args.weak else ""))
    line = {
        "metric": METRIC, "value": r64["value"], "unit": "cell-updates/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r64["ms_per_step"], "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "grid": list(grid), "precision": "fp64",
                   "mode": "cfl 0.4 (dt allreduce each step)" + (", bulk-momentum forcing (O-27)" if channel else ""),
                   "decomposition": f"z-slab x{ws}", "transport": transport,
                   "l2": "inputs larger than L2 (one state = %d MB)" % (5 * grid[0] * grid[1] * grid[2] * 8 // 2**20)},
        "clocks": r64["clocks"],
        "gpu_launches": int(r64["total_launches"]),
        "roofline": flux_roofline(r64, grid, ws, args.steps, "fp64", sm_max),
        "hbm_roofline": {"alg_bytes_per_cell_update": alg_bytes,
                         "achieved_gbs": r64["value"] / ws * alg_bytes / 1e9, "peak_gbs": hbm,
                         "frac": r64["value"] / ws * alg_bytes / 1e9 / hbm, "peak_source": "of measured (MEASURED_PEAKS.json hbm_gbs)"},
        "kernel_ms_per_step": {k: v / args.steps for k, v in r64["ms_k"].items()},
        "aux_ms": r64.get("aux"),
    }
    if transport == "loopback":
        line["config"]["note"] = (f"{ws} slab ranks in one process (loopback group) on "
                                  f"{min(ws, _ndev())} GPU(s): a functional dry run of the N-rank path, not a scaling number")
    if "e2e" in r64:
        line["e2e"] = r64["e2e"]
        line["e2e_sync"] = r64.get("e2e_sync")
    cells = grid[0] * grid[1] * grid[2]
    line["memory"] = {"fp64_bytes": r64["mem_bytes"], "fp64_bytes_per_cell": r64["mem_bytes"] / cells,
                      "note": "device memory allocated by hgks_create (cudaMemGetInfo delta), all ranks; Table 8's "
                              "memory cost (P:1043-1071)"}
    if "fp32" in results:
        r32 = results["fp32"]
        line["memory"].update({"fp32_bytes": r32["mem_bytes"], "fp32_bytes_per_cell": r32["mem_bytes"] / cells,
                               "R_fp": r64["mem_bytes"] / max(1, r32["mem_bytes"])})
        line["fp32"] = {"value": r32["value"], "ms_per_step": r32["ms_per_step"], "clocks": r32["clocks"],
                        "e2e": r32.get("e2e"), "e2e_sync": r32.get("e2e_sync"),
                        "speedup_vs_fp64": r32["value"] / r64["value"],
                        "roofline": flux_roofline(r32, grid, ws, args.steps, "fp32", sm_max),
                        "kernel_ms_per_step": {k: v / args.steps for k, v in r32["ms_k"].items()}}
    if not args.no_cpu and not channel:
        line["cpu_baseline"] = cpu_baseline_block(n, args.cpu_planes, prm["mu"])
    print(json.dumps(line), flush=True)


def _ndev():
    import torch
    return max(1, torch.cuda.device_count())


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hgks", choices=["hgks", "reference"])
    ap.add_argument("--transport", default="nccl", choices=["nccl", "loopback", "nccl-self"],
                    help="nccl: one process per GPU; loopback: N ranks in this process (one GPU suffices); "
                         "nccl-self: one rank with a one-member NCCL communicator (the z halo as NCCL self "
                         "send/recv, the CFL word by NCCL allreduce): the NCCL code path on one GPU")
    ap.add_argument("--n", type=int, default=256, help="TGV grid n^3 (BASELINE config 3: 256)")
    ap.add_argument("--workload", default="tgv", choices=["tgv", "channel"],
                    help="tgv: config 3 (headline); channel: config 4 (H2 128x256x128 unless --channel-grid)")
    ap.add_argument("--channel-grid", default="128,256,128")
    ap.add_argument("--weak", action="store_true", help="weak scaling (config 5 with --n 512): n x n x (n/8 * N)")
    ap.add_argument("--no-fp32", action="store_true")
    ap.add_argument("--only-fp32", action="store_true", help="profiling aid: run only the fp32 leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-planes", type=int, default=4)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    if args.transport == "nccl-self" and args.gpus != 1:
        raise SystemExit("bench.py: --transport nccl-self is a one-rank run (--gpus 1)")
    if args.transport == "nccl" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # the driver launches N > 1 under torch.distributed.run; a bare `--gpus N` re-executes so
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))

    import torch

    if args.transport == "loopback":
        ws = args.gpus
        shared = LoopbackShared(ws)
        outs, errs = [None] * ws, []

        def work(r):
            try:
                outs[r] = measure_rank(args, LoopbackEnv(shared, r, _ndev()))
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
                shared.bar.abort()

        th = [threading.Thread(target=work, args=(r,)) for r in range(ws)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        if outs[0] is not None:
            report(args, outs[0], ws, "loopback")
        return

    import torch.distributed as dist
    ws, rank, local = _dist()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if ws > torch.cuda.device_count():
        raise SystemExit(f"bench.py: {ws} NCCL ranks need {ws} GPUs, {torch.cuda.device_count()} visible "
                         "(use --transport loopback for a one-GPU dry run)")
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = measure_rank(args, NcclEnv(dist, ws, rank, local, self_comm=args.transport == "nccl-self"))
    if out is not None:
        report(args, out, ws, "nccl" if ws > 1 else ("nccl (one-member communicator)" if args.transport == "nccl-self"
                                                      else "none (1 rank)"))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
