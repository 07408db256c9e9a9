#!/usr/bin/env python
"""Benchmark of the FKS hot path on B200.

One "step" = one fks_step over the whole workload: exact transport gather (a1) + forward transform (a2) +
T+1 separated terms (a3-a5) + back transform and explicit Euler write-back (a6-a7) + generic-cell
bookkeeping (a8).  Default workload: BASELINE.json configs[3] (c3: 32^3 cells x 32^3 velocities, hard
spheres, M = 32), the configuration the headline target is quoted on.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

N > 1 is launched by torchrun: every rank runs its own c3 box (independent cells, no data-path collective:
weak scaling); time = max over ranks of the CUDA-event time; rank 0 prints ONE JSON line.
`--impl reference` times the CPU oracle (tests' reference implementation) on a bounded sample of the same
workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_UNITS_PER_SM = 64          # DFMA lanes per SM per clock (B200, sm_100a)
N_SMS = 148


def flops_per_cell(N: int, P: int, T: int) -> dict:
    """Algorithmic FLOPs per cell: conventional FFT counts (5 n log2 n per
    complex length-n transform, 2.5 for real) of the pruned Galerkin computation + element-wise work."""
    K = N - 1
    lg = math.log2
    fwd = 2.5 * N ** 3 * lg(N ** 3)
    inv_term = 5 * P * lg(P) * (K * K + K * P + P * P)
    elem_term = 4 * K ** 3 + 2 * P ** 3
    back = 2.5 * P * lg(P) * (P * P + P * K + K * K) + 2.5 * N ** 3 * lg(N ** 3)
    hot = (T + 1) * (inv_term + elem_term)
    return {"forward": fwd, "hot": hot, "back": back, "total": fwd + hot + back}


def fp64_peak_tflops(sm_mhz: float) -> float:
    return N_SMS * FP64_UNITS_PER_SM * 2 * sm_mhz * 1e6 / 1e12


# ------------------------------------------------------------------------------------------------------
# clocks during the timed region
# ------------------------------------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_bench_{os.getpid()}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            # let nvidia-smi initialise (first sample written) before the timed region starts: its start-up
            # stalled the host thread by tens of ms, which doubled the measured time of short (c1) runs
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 2.0:
                self.fh.flush()
                if os.path.getsize(self.path) > 0:
                    break
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[2]) for r in rows)}


# ------------------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline / --impl reference)
# ------------------------------------------------------------------------------------------------------

def oracle_threads() -> int:
    """Host threads the C++ oracle's std::thread pool uses (every core this process may run on)."""
    from oracle import cpp_oracle as co
    return co.default_threads()


def blas_threads() -> int:
    """Threads the numpy (BLAS) oracle may use: the BGK leg still times the numpy oracle."""
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return os.cpu_count() or 1


def host_cpu() -> dict:
    """nproc and CPU model of the host the oracle is timed on."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "affinity": oracle_threads(), "model": model}


def time_oracle(cfg, budget_s: float, max_cells: int = 256, min_batches: int = 1) -> dict:
    """The plain C++17 oracle (oracle/cpp, std::thread pool over cells, naive per-axis DFTs; BJ.north_star) on
    sampled cells of the workload: collision + Euler per sampled cell (the transport is a permutation of the
    inputs), one batch of `threads` cells at a time, until `budget_s` has elapsed."""
    from oracle import cpp_oracle as co
    from paper_1701_01608_b200 import inputs
    tb = co.build_tables(cfg.N, cfg.L, M=cfg.M, M_r=cfg.M_r, kernel=cfg.kernel)
    thr = co.default_threads()
    cells = inputs.sample_cells(cfg, min(max_cells, cfg.n_cells), seed=5)
    f = inputs.make_f(cfg, cells=cells).numpy()
    t0 = time.perf_counter()
    n = nb = 0
    while n < len(f):
        batch = f[n:n + thr]
        co.euler(batch, co.collision_batch(batch, tb, threads=thr), cfg.coll_scale)
        n += len(batch)
        nb += 1
        if nb >= min_batches and time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"cells": n, "seconds": dt, "value": n * cfg.N ** 3 / dt, "threads": thr}


# ------------------------------------------------------------------------------------------------------
# BGK workload: fks_bgk_step = transport gather + moments + BGK relaxation, one fused
# kernel; HBM-bound (algorithmic traffic 16 B per cell-velocity point: read f_in once, write f_out once)
# ------------------------------------------------------------------------------------------------------

BGK_NU = 10.0  # ν = 1/τ with τ = 0.1, the paper's BGK Sod runs


def hbm_peak_gbs() -> tuple:
    try:
        return float(json.load(open(MEASURED_PEAKS))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except Exception:
        return 7700.0, "nominal 7.7 TB/s (MEASURED_PEAKS.json unavailable)"


def time_oracle_bgk(cfg, budget_s: float, nu_dt: float, max_cells: int = 1024) -> dict:
    import numpy as np  # noqa: F401
    from oracle import fks_oracle as o
    from paper_1701_01608_b200 import inputs
    cells = inputs.sample_cells(cfg, min(max_cells, cfg.n_cells), seed=7)
    f = inputs.make_f(cfg, cells=cells).numpy()
    t0 = time.perf_counter()
    n = 0
    for fc in f:  # transport is a permutation of the inputs: relaxation of the sampled cells
        fc + nu_dt * (o.local_maxwellian(fc, cfg.N, cfg.L) - fc)
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"cells": n, "seconds": dt, "value": n * cfg.N ** 3 / dt}


def bgk_traffic(cfg):
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "r01j_bgk_step_traffic.json")))
        return tj["dram_bytes_per_cell"] * cfg.n_cells if cfg.N == 32 else None
    except Exception:
        return None


def run_bgk(args):
    from paper_1701_01608_b200 import dist as D
    from paper_1701_01608_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    ws, rank, local = D.world()
    metric = "fp64 BGK FKS step (transport + moments + relaxation) cell·velocity-points/s; fraction of HBM roofline"
    unit = "cell·vp/s"
    dt_over_dx = cfg.cfl_num / cfg.cfl_den / cfg.L  # Δt = c Δx / L
    nu_dt = BGK_NU * dt_over_dx / cfg.shape[0]
    workload = {"workload": f"{cfg.name} box, BGK operator: {cfg.shape[0]}x{cfg.shape[1]}x{cfg.shape[2]} cells x "
                            f"{cfg.N}^3 velocities, fks_bgk_step (transport c={cfg.cfl_num}/{cfg.cfl_den}, "
                            f"nu={BGK_NU}, nu*dt={nu_dt:.6g})",
                "config": cfg.name, "n_cells": cfg.n_cells, "N": cfg.N,
                "l2": "inputs larger than L2 (f is %.2f GB per copy)" % (cfg.n_cells * cfg.N ** 3 * 8 / 1e9)}
    if args.impl == "reference":
        if rank != 0:
            return
        times, cells = [], 0
        per_step = max(2.0, min(args.cpu_seconds, 120.0 / max(1, args.steps + args.warmup)))
        for i in range(args.warmup + args.steps):
            r = time_oracle_bgk(cfg, per_step, nu_dt)
            if i >= args.warmup:
                times.append(r["seconds"])
                cells += r["cells"]
        val = cells * cfg.N ** 3 / sum(times)
        print(json.dumps({"impl": "reference", "metric": metric, "value": val, "unit": unit, "n_gpus": args.gpus,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "config": workload,
                          "cpu_baseline": {"value": val, "unit": unit, "cores": blas_threads(), "kind": "oracle",
                                           "sample": f"{cells} cells of {cfg.name} (BGK relaxation per sampled cell)"},
                          "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch
    import torch.distributed as dist
    from paper_1701_01608_b200 import binding as B
    from paper_1701_01608_b200 import inputs
    if ws > 1:
        torch.cuda.set_device(local % torch.cuda.device_count())
        # FKS_BENCH_BACKEND=gloo only to exercise the multi-rank flow where the ranks share one GPU (no timing claim)
        dist.init_process_group(os.environ.get("FKS_BENCH_BACKEND", "nccl"), init_method="env://")
    dev = torch.device("cuda", local % torch.cuda.device_count() if ws > 1 else 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    fa = inputs.make_f(cfg, device=dev, seed=D.rank_seed(rank))
    fb = torch.empty_like(fa)
    col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)

    def barrier():
        if ws > 1:
            dist.barrier()

    bufs = [fa, fb]
    for i in range(args.warmup):
        col.bgk_step(bufs[i % 2], bufs[(i + 1) % 2], nu_dt)
    torch.cuda.synchronize()
    barrier()
    n0 = col.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clk:
        torch.cuda.synchronize()
        barrier()
        e0.record(stream)
        for i in range(args.steps):
            col.bgk_step(bufs[(args.warmup + i) % 2], bufs[(args.warmup + i + 1) % 2], nu_dt)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = col.launches() - n0
    ms_step = D.max_over_ranks(e0.elapsed_time(e1), dev) / args.steps
    value = D.weak_value(cfg.n_cells, cfg.N ** 3, ws, ms_step)
    nbytes = cfg.n_cells * cfg.N ** 3 * 8
    achieved = 2 * nbytes / (ms_step / 1e3) / 1e9
    peak, peak_note = hbm_peak_gbs()

    e2e = None
    if not args.no_e2e:  # pinned host -> device, the fused step, device -> pinned host, all timed
        hin = torch.empty(fa.shape, dtype=torch.float64, pin_memory=True)
        hout = torch.empty_like(hin, pin_memory=True)
        hin.copy_(fa)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            fa.copy_(hin, non_blocking=True)
            col.bgk_step(fa, fb, nu_dt)
            hout.copy_(fb, non_blocking=True)
        torch.cuda.synchronize()
        dt = D.max_over_ranks(time.perf_counter() - t0, dev)
        e2e = {"value": cfg.n_cells * ws * cfg.N ** 3 * args.e2e_steps / dt, "unit": unit,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": args.e2e_steps,
               "api": "torch pinned H2D + Collision.bgk_step (fks_bgk_step) + D2H"}
        del hin, hout
    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    cpu = time_oracle_bgk(cfg, min(args.cpu_seconds, 10.0), nu_dt)
    print(json.dumps({
        "metric": metric, "value": value, "unit": unit, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": bgk_traffic(cfg),
                     "traffic_note": "dram__bytes_read+write per launch from profiles/r01j_bgk_step_traffic.json "
                                     "(ncu --set full of this kernel on this workload)",
                     "kernel": "macro_kernel<BGK_STEP> (fused transport gather + moments + relaxation)",
                     "bytes_per_cell_vp": 16, "peak_note": peak_note},
        "clocks": clk.summary(), "gpu_launches": launches, "e2e": e2e,
        "cpu_baseline": {"value": cpu["value"], "unit": unit, "cores": blas_threads(), "kind": "oracle",
                         "sample": f"{cpu['cells']} sampled cells of {cfg.name}, BGK relaxation, {cpu['seconds']:.1f} s"},
    }))
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--decomposed", action="store_true",
                    help="N ranks run ONE periodic box of N x 32 x-planes, slab-decomposed in x (fks_step_slab: the "
                         "transport gathers across slab boundaries from the neighbours' memory over NVLink, one "
                         "barrier per step) instead of N independent boxes")
    ap.add_argument("--no-decomposed-extra", action="store_true",
                    help="N > 1: skip the extra slab-decomposed measurement reported under 'decomposed'")
    ap.add_argument("--workload", default="boltzmann", choices=["boltzmann", "bgk"],
                    help="bgk: the BGK-operator FKS step (SURVEY §8(f) NEXT-3; HBM-bound) on the same config")
    args = ap.parse_args()
    if args.workload == "bgk":
        return run_bgk(args)

    from paper_1701_01608_b200 import dist as D
    from paper_1701_01608_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    ws, rank, local = D.world()
    metric = "fp64 Q(f,f) cell·velocity-points/s on 1 B200; fraction of FP64/HBM roofline"
    unit = "cell·vp/s"
    workload = {"workload": f"{cfg.name}: {cfg.shape[0]}x{cfg.shape[1]}x{cfg.shape[2]} cells x {cfg.N}^3 velocities, "
                            f"{'hard spheres' if cfg.kernel == 0 else 'Maxwell molecules'}, M={cfg.M}, fks_step "
                            f"(transport c={cfg.cfl_num}/{cfg.cfl_den} + collision + Euler, s={cfg.coll_scale:.6g})",
                "config": cfg.name, "n_cells": cfg.n_cells, "N": cfg.N, "M": cfg.M,
                "l2": "inputs larger than L2 (f is %.2f GB per copy)" % (cfg.n_cells * cfg.N ** 3 * 8 / 1e9)}

    if args.impl == "reference":
        if rank != 0:
            return
        times = []
        cells = 0
        per_step = max(2.0, min(args.cpu_seconds, 120.0 / max(1, args.steps + args.warmup)))
        for i in range(args.warmup + args.steps):
            r = time_oracle(cfg, per_step, max_cells=oracle_threads())
            if i >= args.warmup:
                times.append(r["seconds"])
                cells += r["cells"]
        val = cells * cfg.N ** 3 / sum(times)
        line = {"impl": "reference", "metric": metric, "value": val, "unit": unit, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": workload,
                "cpu_baseline": {"value": val, "unit": unit, "cores": oracle_threads(), "kind": "oracle",
                                 "host": host_cpu(),
                                 "sample": f"{cells} cells of {cfg.name} (collision+Euler per sampled cell, C++ "
                                           f"oracle, one batch of {oracle_threads()} cells per step), "
                                           f"{args.steps} steps"},
                "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    from paper_1701_01608_b200 import binding as B
    from paper_1701_01608_b200 import inputs

    if ws > 1:
        torch.cuda.set_device(local % torch.cuda.device_count())
        # FKS_BENCH_BACKEND=gloo only to exercise the multi-rank flow where the ranks share one GPU (no timing claim)
        dist.init_process_group(os.environ.get("FKS_BENCH_BACKEND", "nccl"), init_method="env://")
    dev = torch.device("cuda", local % torch.cuda.device_count() if ws > 1 else 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)

    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    P, T = col.info["P"], col.info["T"]
    fa = inputs.make_f(cfg, device=dev, seed=D.rank_seed(rank))
    fb = torch.empty_like(fa)
    col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
    s = cfg.coll_scale

    def barrier():
        if ws > 1:
            dist.barrier()

    bufs = [fa, fb]
    stepper = None
    if args.decomposed:  # one global box, x-slab per rank (rank r's own c3 box is its slab)
        dom = D.SlabDomain(cfg.shape[0] * ws, cfg.shape[1], cfg.shape[2], rank, ws)
        stepper = D.SlabStepper(col, dom, fa, fb, cfg.cfl_num, cfg.cfl_den, barrier=D.stream_barrier(dev))
        workload["workload"] += f"; decomposed: one {cfg.shape[0] * ws}x{cfg.shape[1]}x{cfg.shape[2]} box, x-slabs"
        workload["parallelism"] = f"x-slabs over {ws} ranks, peer-memory transport gather"

    def one_step(i):
        if stepper is not None:
            stepper.step(s)
        else:
            col.step(bufs[i % 2], bufs[(i + 1) % 2], s)

    # W warm-up steps; on one rank at least 0.3 s of them, so that tiny workloads (c0) are timed at full clocks
    # (several ranks keep exactly W: the decomposed step has a collective per step)
    t_w = time.perf_counter()
    nw = 0
    while nw < args.warmup or (ws == 1 and time.perf_counter() - t_w < 0.3):
        one_step(nw)
        nw += 1
        if nw >= args.warmup:
            torch.cuda.synchronize()
    args.warmup = nw
    torch.cuda.synchronize()
    barrier()
    B.fks_profile(col.h, True)
    B.fks_profile_read(col.h)  # reset
    n0 = col.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clk:
        torch.cuda.synchronize()
        barrier()
        e0.record(stream)
        for i in range(args.steps):
            one_step(args.warmup + i)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms_total = e0.elapsed_time(e1)
    launches = col.launches() - n0
    ph_ms, ph_cnt = B.fks_profile_read(col.h)
    B.fks_profile(col.h, False)
    ms_total = D.max_over_ranks(ms_total, dev)
    ms_step = ms_total / args.steps
    cells_all = cfg.n_cells * ws
    value = D.weak_value(cfg.n_cells, cfg.N ** 3, ws, ms_step)

    # roofline of the dominant kernel (the term loop / hot kernel, phase 2)
    fl = flops_per_cell(cfg.N, P, T)
    hot_ms = ph_ms[2] / max(1, ph_cnt[2])
    cells_per_launch = cfg.n_cells * args.steps / max(1, ph_cnt[2])
    achieved = fl["hot"] * cells_per_launch / (hot_ms / 1e3) / 1e12
    clocks = clk.summary()
    # FP64 unit-count peak at the SM clock observed under load (median of the samples), max clock if unsampled
    sm_used = clocks.get("sm_mhz") or 1965.0
    peak = fp64_peak_tflops(sm_used)
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture of this kernel (per cell,
    # scaled to this run's cells per launch); null when no capture of the current kernel is committed
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", f"r02_hot_kernel_traffic_N{cfg.N}.json")
    if os.path.exists(tpath) and col.info.get("path") == 2:
        try:
            tj = json.load(open(tpath))
            traffic = tj["dram_bytes_per_cell"] * cells_per_launch
            traffic_src = f"profiles/{os.path.basename(tpath)}: {tj.get('source', '')}"
        except Exception:
            traffic = None

    # N > 1: the same workload once more through the slab-decomposed path (one global box of ws x 32 x-planes,
    # transport gathering across slab boundaries from the neighbours' memory, interior planes before the
    # per-step barrier): the multi-GPU data path the paper's MPI FKS exercises
    decomposed = None
    if ws > 1 and not args.decomposed and not args.no_decomposed_extra:
        try:
            dom = D.SlabDomain(cfg.shape[0] * ws, cfg.shape[1], cfg.shape[2], rank, ws)
            dcol = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
            dst = D.SlabStepper(dcol, dom, fa, fb, cfg.cfl_num, cfg.cfl_den, barrier=D.stream_barrier(dev))
            for _ in range(min(args.warmup, 2)):
                dst.step(s)
            torch.cuda.synchronize()
            barrier()
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            for _ in range(args.steps):
                dst.step(s)
            d1.record(stream)
            torch.cuda.synchronize()
            barrier()
            dms = D.max_over_ranks(d0.elapsed_time(d1), dev) / args.steps
            decomposed = {"value": D.weak_value(cfg.n_cells, cfg.N ** 3, ws, dms), "unit": unit, "ms_per_step": dms,
                          "box": f"{cfg.shape[0] * ws}x{cfg.shape[1]}x{cfg.shape[2]} cells, x-slab of "
                                 f"{dom.nx_local} planes per rank, halo {dst.H}", "scaling": "weak",
                          "api": "fks_step_slab_range (interior planes, barrier, boundary planes)"}
            del dst, dcol
        except Exception as ex:  # report, never lose the main line
            decomposed = {"error": f"{type(ex).__name__}: {ex}"[:300]}

    # end to end through the host-buffer C-ABI call (pinned host memory, copies inside the timed region)
    e2e = None
    if not args.no_e2e and not args.decomposed:
        hin = torch.empty(fa.shape, dtype=torch.float64, pin_memory=True)
        hout = torch.empty_like(hin, pin_memory=True)
        hin.copy_(fa)
        col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
        B.fks_step_host(col.h, hin, hout, s)  # warm-up (allocates staging)
        barrier()
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            B.fks_step_host(col.h, hin if i % 2 == 0 else hout, hout if i % 2 == 0 else hin, s)
        dt = D.max_over_ranks(time.perf_counter() - t0, dev)
        nbytes = cfg.n_cells * cfg.N ** 3 * 8
        e2e = {"value": cells_all * cfg.N ** 3 * args.e2e_steps / dt, "unit": unit,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": args.e2e_steps,
               "api": "fks_step_host (pinned host buffers)"}
        # the collision operator alone through the host-buffer call (BASELINE's Q(f,f) metric end to end)
        B.fks_collision_batch_host(col.h, hin, hout, cfg.n_cells)  # warm-up
        barrier()
        t0 = time.perf_counter()
        B.fks_collision_batch_host(col.h, hin, hout, cfg.n_cells)
        dt = D.max_over_ranks(time.perf_counter() - t0, dev)
        e2e["collision_only"] = {"value": cells_all * cfg.N ** 3 / dt, "unit": unit,
                                 "api": "fks_collision_batch_host (pinned host buffers)"}
        del hin, hout

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return

    cpu = time_oracle(cfg, args.cpu_seconds)
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_note": ("dram__bytes_read+write per launch, " + traffic_src +
                                      " (one ncu --set full capture of this kernel), scaled to cells per launch")
                                     if traffic_src else "no committed ncu capture of this kernel",
                     "kernel": ("term loop (a3-a5): " + ("hot_kernel_v4, 12-CTA teams" if cfg.N == 32 else
                                "small_term_kernel, one CTA per (cell, z-class, term chunk)")),
                     "flop_per_cell": fl["hot"], "cells_per_launch": cells_per_launch, "ms_per_launch": hot_ms,
                     "timing_note": ("CUDA events on the term-loop kernel's own (high-priority) stream, each launch "
                                     "running beside the chunk pipeline's forward / back transforms on the SMs its "
                                     "teams leave free (DESIGN.md §5); run alone it is ~0.5 % faster "
                                     "(FKS_NO_PIPELINE=1)") if (cfg.N == 32 and ph_cnt[2] > args.steps
                                                               and not os.environ.get("FKS_NO_PIPELINE"))
                                    else "CUDA events on the launching stream",
                     "frac_of_measured_dfma": achieved / 36.66,
                     "peak_at_max_clock": fp64_peak_tflops(1965.0),
                     # the N = 32 kernel is sensitive to how its warp roles phase-lock; the shipped
                     # build runs at about 375 ns per cell and term (137 ms per 10 923-cell c3 launch): record
                     # whether this run landed there or on a slower point
                     "operating_point": (("fast" if hot_ms * 1e6 / (cells_per_launch * (T + 1)) < 395.0 else "slow")
                                         if cfg.N == 32 and col.info.get("path") == 2 else None),
                     "ns_per_cell_term": hot_ms * 1e6 / (cells_per_launch * (T + 1)),
                     "peak_note": f"FP64 DFMA unit counts: 148 SM x 64 lanes x 2 flop x {sm_used:.0f} MHz (median SM "
                                  "clock sampled under load); measured DFMA 36.66 TF/s with 16 warps per SM "
                                  "(profiles/r02_dmma_dfma_mix.jsonl; 33.6 with 8 chains in r01_box_microbench)"},
        "whole_step": {"flop_per_cell": fl["total"],
                       "tflops": fl["total"] * cells_all / ws / (ms_step / 1e3) / 1e12,
                       "frac_of_fp64_peak": fl["total"] * cells_all / ws / (ms_step / 1e3) / 1e12 / peak,
                       "hbm_bytes_per_cell": 16 * cfg.N ** 3},
        "phases_ms_per_step": {"transport": ph_ms[0] / args.steps, "forward": ph_ms[1] / args.steps,
                               "term_loop": ph_ms[2] / args.steps, "back": ph_ms[3] / args.steps},
        "phases_note": ("chunk pipeline: the forward / back transforms of neighbouring workspace chunks run on a "
                        "low-priority stream beside the term-loop launches (on the 4 SMs the 12-CTA teams leave "
                        "free and in each launch's tail), so their intervals overlap the term loop and do not add "
                        "up to ms_per_step") if (cfg.N == 32 and ph_cnt[2] > args.steps
                                                 and not os.environ.get("FKS_NO_PIPELINE")) else None,
        "path": {1: "generic", 2: "fast"}.get(col.info.get("path"), None),
        "fast_layout": {"ctas_per_cell": col.info.get("ctas_per_cell"), "concurrent_cells": col.info.get("concurrent_cells")},
        "clocks": clocks, "gpu_launches": launches, "e2e": e2e, "decomposed": decomposed,
        "cpu_baseline": {"value": cpu["value"], "unit": unit, "cores": cpu["threads"], "kind": "oracle",
                         "host": host_cpu(),
                         "sample": f"{cpu['cells']} sampled cells of {cfg.name}, collision+Euler, "
                                   f"{cpu['seconds']:.1f} s (plain C++17 fp64 oracle, naive per-axis DFTs, "
                                   f"std::thread pool of {cpu['threads']} over cells)"},
    }
    print(json.dumps(line))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
