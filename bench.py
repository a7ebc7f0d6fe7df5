#!/usr/bin/env python
"""bench.py — HGKS S2O4 step throughput on B200 (BASELINE.json metric: cell-updates/s, TGV 256^3).

One "step" = one full two-stage S2O4 step (A0..A8 of SURVEY.md §8(a)) over the whole grid.
Launch: python bench.py [--gpus N --steps K --warmup W]; N > 1 under torch.distributed.run
(one rank per GPU, NCCL halos along z).  --impl reference times the plain CPU oracle instead.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/s"
# FP64 peak of B200 derived from unit counts: 148 SMs x 64 FP64 FMA/clk
# x 2 flop x clocks.max.sm (1965 MHz, MEASURED_PEAKS.json sm_max_mhz)
N_SM, FP64_FMA_PER_CLK = 148, 64


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


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


def _flop_table():
    path = os.path.join(ROOT, "profiles", "flux_flops.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def cpu_baseline(n: int, planes: int, mu: float, dx, stage_count: int = 2):
    """Oracle (CPU, all host cores via OpenMP) on a bounded sample of the same TGV workload:
    the operator L, d_t L of `planes` z-planes of the n^3 field (true neighbour ghosts), once
    per stage.  Returns (cell-updates/s, cores, seconds, sample description)."""
    from oracle import oracle as O
    from paper_2207_01173_b200 import inputs
    # ghosted block: z planes -3 .. planes+2 of the periodic n^3 field, x/y ghosts by wrap
    zidx = np.arange(-3, planes + 3) % n
    blk_z = np.concatenate([inputs.tgv(n, z_begin=int(z), nz_local=1)[0] for z in zidx], axis=1)
    w = np.arange(-3, n + 3) % n
    blk = np.ascontiguousarray(blk_z[:, :, w][:, :, :, w])
    gas = O.make_gas(mu=mu)
    dummy = np.zeros((5, planes, n, n))
    t0 = time.perf_counter()
    for _ in range(stage_count):
        O.operator(gas, dummy, dx, 1e-3, qg=blk)
    sec = time.perf_counter() - t0
    cells = n * n * planes
    return cells / sec, O.num_threads(), sec, f"oracle operator on {n}x{n}x{planes} z-planes of TGV {n}^3, x{stage_count} stages"


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    n = args.n
    prm = __import__("paper_2207_01173_b200.inputs", fromlist=["tgv_params"]).tgv_params()
    dx = (2 * math.pi / n,) * 3
    planes = 1
    times = []
    for i in range(args.warmup + args.steps):
        v, cores, sec, sample = cpu_baseline(n, planes, prm["mu"], dx)
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hgks", choices=["hgks", "reference"])
    ap.add_argument("--n", type=int, default=256, help="TGV grid n^3 (BASELINE config 3: 256)")
    ap.add_argument("--workload", default="tgv", choices=["tgv", "channel"],
                    help="tgv: config 3 (headline); channel: config 4 (H2 128x256x128 unless --channel-grid)")
    ap.add_argument("--channel-grid", default="128,256,128")
    ap.add_argument("--weak", action="store_true", help="weak scaling: n x n x (n/8 * N) per job")
    ap.add_argument("--no-fp32", action="store_true")
    ap.add_argument("--only-fp32", action="store_true", help="profiling aid: run only the fp32 leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-planes", type=int, default=4)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2207_01173_b200 import hgks as H
    from paper_2207_01173_b200 import inputs

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = args.n
    nz = (n // 8) * ws if args.weak else n
    grid = (n, n, nz)
    prm = inputs.tgv_params()
    channel = args.workload == "channel"
    if channel:
        grid = tuple(int(x) for x in args.channel_grid.split(","))
        chp = inputs.channel_params()
    nccl_id = None
    if ws > 1:
        obj = [H.hgks_get_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if ws == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    lo, hi = (-math.pi,) * 3, (math.pi,) * 3  # weak mode: same box, nz = n/8 * N planes (anisotropic dz)

    def make_solver(precision):
        if channel:  # config 4: walls in y, tanh mesh, power-law mu, Pr = 0.7
            return H.Solver(grid, chp["lo"], chp["hi"], mu=chp["mu_w"], mu_law=H.HGKS_MU_POWER, T_ref=chp["T_w"],
                            omega=chp["omega"], prandtl=chp["prandtl"], T_wall=chp["T_w"],
                            bc=(H.HGKS_PERIODIC, H.HGKS_WALL_ISOTHERMAL, H.HGKS_PERIODIC),
                            stretch=(H.HGKS_UNIFORM, H.HGKS_TANH, H.HGKS_UNIFORM), stretch_b=(0.0, chp["b_g"], 0.0),
                            cfl=0.4, precision=precision, rank=rank, nranks=ws, device=local, nccl_id=nccl_id,
                            stream=stream.cuda_stream,
                            # constant bulk momentum rho_b U_b = 1 (units of the channel, O-27)
                            force_mode=H.HGKS_FORCE_BULK, force=0.0, force_target=1.0)
        return H.Solver(grid, lo, hi, mu=prm["mu"], cfl=0.4, precision=precision, rank=rank, nranks=ws,
                        device=local, nccl_id=nccl_id, stream=stream.cuda_stream)

    def local_field(s):
        if channel:
            return inputs.channel(grid, z_begin=s.z0, nz_local=s.nz_local)[0]
        # TGV on [-pi, pi]^3 with this rank's z planes
        q, _ = inputs.tgv(grid, z_begin=s.z0, nz_local=s.nz_local)
        return q

    results = {}
    for prec_name, prec in (("fp64", H.HGKS_FP64), ("fp32", H.HGKS_FP32)):
        if prec_name == "fp32" and args.no_fp32:
            continue
        if prec_name == "fp64" and args.only_fp32:
            continue
        s = make_solver(prec)
        q = local_field(s)
        qd = torch.from_numpy(q).cuda()
        s.set_state(qd)
        s.step(args.warmup)
        barrier()
        H.hgks_profile_enable(s.ctx, True)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            barrier()
            ev0.record(stream)
            s.step(args.steps)
            ev1.record(stream)
            barrier()
        ms_local = ev0.elapsed_time(ev1)
        ms_k, launches, total_launches = H.hgks_profile_read(s.ctx)
        H.hgks_profile_enable(s.ctx, False)
        ms = max_over_ranks(ms_local)
        cells = grid[0] * grid[1] * grid[2]
        rate = cells * args.steps / (ms / 1000.0)
        res = dict(ms_per_step=ms / args.steps, value=rate, clocks=clk.summary(), ms_k=ms_k, launches=launches,
                   total_launches=total_launches, t=s.t)
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
            torch.cuda.synchronize()
            aux[name + "_ms"] = a0.elapsed_time(a1) / 3
        res["aux"] = aux
        # e2e through the public API with host buffers (pinned): H2D state, step, D2H state per step
        if not args.no_e2e:
            qh = torch.from_numpy(q).pin_memory()
            qo = torch.empty_like(qh).pin_memory()
            barrier()
            t0 = time.perf_counter()
            e_ev0, e_ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e_ev0.record(stream)
            e_steps = max(2, min(args.steps, 5))
            for _ in range(e_steps):
                s.set_state(qh.numpy())
                s.step(1)
                s.get_state(qo.numpy())
            e_ev1.record(stream)
            barrier()
            e_ms = max_over_ranks(e_ev0.elapsed_time(e_ev1))
            res["e2e"] = {"value": cells * e_steps / (e_ms / 1000.0), "unit": "cell-updates/s",
                          "h2d_bytes_per_step": int(q.nbytes) * ws, "d2h_bytes_per_step": int(q.nbytes) * ws,
                          "steps": e_steps, "wall_s": time.perf_counter() - t0}
        s.close()
        del qd
        torch.cuda.empty_cache()
        results[prec_name] = res

    if rank != 0 or args.only_fp32:
        if ws > 1:
            dist.destroy_process_group()
        return
    r64 = results["fp64"]
    flux_ms = sum(r64["ms_k"][k] for k in ("flux_x", "flux_y", "flux_z"))
    flux_launches = sum(r64["launches"][k] for k in ("flux_x", "flux_y", "flux_z"))
    ftab = _flop_table()
    clk = r64["clocks"]
    peaks = _peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak_tflops = N_SM * FP64_FMA_PER_CLK * 2 * sm_max * 1e6 / 1e12
    cells_local = grid[0] * grid[1] * grid[2] // ws
    roof = {"bound": "alu", "kernel": "flux_kernel<double,DIR,STAGE> (x,y,z faces, both stages)",
            "peak": peak_tflops, "unit": "TFLOP/s",
            "peak_source": f"derived: {N_SM} SMs x {FP64_FMA_PER_CLK} FP64 FMA/clk x 2 x {sm_max:.0f} MHz (DESIGN.md)",
            # share of the step's wall time (the reconstruction kernels overlap on a second stream, so
            # the per-class event sums exceed the wall time; compare with the serialised ncu share)
            "flux_share_of_step": flux_ms / (r64["ms_per_step"] * args.steps) if r64["ms_per_step"] else None,
            "avg_launch_ms": flux_ms / flux_launches if flux_launches else None, "traffic": None}
    if ftab:
        # executed FP64 flops per face per stage (ncu SASS count, profiles/flux_flops.json)
        gx, gy, gzl = grid[0], grid[1], grid[2] // ws
        faces = 3 * cells_local + gy * gzl + gx * gzl + gx * gy  # x, y, z faces of one rank's slab
        flops_step = faces * (ftab["flop_per_face_stage1"] + ftab["flop_per_face_stage2"])
        achieved = flops_step * args.steps / (flux_ms / 1000.0) / 1e12
        roof.update(achieved=achieved, frac=achieved / peak_tflops, flop_source=ftab.get("source"),
                    traffic=ftab.get("dram_bytes_per_launch"))
    hbm = float(peaks.get("hbm_gbs", 6542.4))
    alg_bytes = 240.0  # fp64 bytes per cell-update
    line = {
        "metric": METRIC, "value": r64["value"], "unit": "cell-updates/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r64["ms_per_step"], "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": ("channel_" + "x".join(map(str, grid))) if channel else (f"tgv{n}" + ("_weak" if args.weak else "")),
                   "grid": list(grid), "precision": "fp64",
                   "mode": "cfl 0.4 (dt allreduce each step)" + (", bulk-momentum forcing (O-27)" if channel else ""),
                   "decomposition": f"z-slab x{ws}",
                   "l2": "inputs larger than L2 (one state = %d MB)" % (5 * grid[0] * grid[1] * grid[2] * 8 // 2**20)},
        "clocks": clk,
        "gpu_launches": int(r64["total_launches"]),
        "roofline": roof,
        "hbm_roofline": {"alg_bytes_per_cell_update": alg_bytes,
                         "achieved_gbs": r64["value"] / ws * alg_bytes / 1e9, "peak_gbs": hbm,
                         "frac": r64["value"] / ws * alg_bytes / 1e9 / hbm},
        "kernel_ms_per_step": {k: v / args.steps for k, v in r64["ms_k"].items()},
        "aux_ms": r64.get("aux"),
    }
    if "e2e" in r64:
        line["e2e"] = r64["e2e"]
    if "fp32" in results:
        r32 = results["fp32"]
        line["fp32"] = {"value": r32["value"], "ms_per_step": r32["ms_per_step"], "clocks": r32["clocks"],
                        "e2e": r32.get("e2e"), "speedup_vs_fp64": r32["value"] / r64["value"],
                        "kernel_ms_per_step": {k: v / args.steps for k, v in r32["ms_k"].items()}}
    if not args.no_cpu and not channel:
        v, cores, sec, sample = cpu_baseline(n, args.cpu_planes, prm["mu"], (2 * math.pi / n,) * 3)
        line["cpu_baseline"] = {"value": v, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
                                "sample": sample, "seconds": sec}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
