#!/usr/bin/env python
"""Benchmark: FMM mat-vecs/s of relaxed GMRES at N panels (BASELINE.json configs[1] = cfg2).

One step = one relaxed-GMRES solve of cfg2 (icosphere L5, 20480 panels, Laplace
2nd kind, 3 seeded interior charges, theta 0.5, n_crit 128, tol 1e-6, p 12 -> 3,
unrestarted) with b resident in HBM; value = mat-vecs (applies) done / device
time, whole job.  ``e2e`` is the same metric through the public Python API
(``solver.solve`` on a host pinned b, result read back to the host).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) the same solve is partitioned over the N GPUs (strong
scaling): each rank owns a work-balanced range of target and source leaves,
leaf multipoles and result slices are exchanged with NCCL all-gathers, GMRES
runs replicated; device time is the max over ranks.  ``--impl reference``
times the CPU oracle port of the reference path (oracle/fmm_oracle.py) on the
host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_NAME = "cfg2"
P2P_FLOPS_PER_INTERACTION = {"laplace_second": 18, "laplace_first": 11, "stokes": 29}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=CONFIG_NAME)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload_desc(cfg, mesh):
    return {
        "workload": f"{cfg.name}: {mesh.n_panels}-panel icosphere, {cfg.formulation}, "
                    f"{cfg.n_charges} seeded interior charges, theta {cfg.theta}, n_crit {cfg.n_crit}, "
                    f"relaxed GMRES tol {cfg.tol:g}, p {cfg.p_initial}->{cfg.p_min}, unrestarted",
        "panels": mesh.n_panels,
        "unknowns": mesh.n_panels * (3 if cfg.formulation == "stokes" else 1),
        "gauss_points_far": 4,
        "near_rule": "19-pt degree 9 + 32-node polar singular",
        "step": "one relaxed GMRES solve (b resident in HBM)",
        "l2": "256 MiB buffer written between timed steps (L2 flush)",
    }


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = list(csv.reader(io.StringIO(open(self.path).read())))
        os.unlink(self.path)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows[1:]:
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1].split()[0]))
                smax.append(float(r[2].split()[0]))
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip() == "Active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU (oracle) legs
def cpu_threads():
    n = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(n)
    except Exception:
        pass
    return n


def cpu_baseline_sample(cfg, mesh, b):
    """Oracle port (oracle/fmm_oracle.py): one relaxed GMRES solve of the same config."""
    from oracle import fmm_oracle as O

    cores = cpu_threads()
    op = O.OracleOperator(mesh, cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
    t0 = time.perf_counter()
    r = O.gmres(op.apply, b, O.RelaxationSchedule(cfg.p_initial, cfg.p_min, cfg.tol, True), cfg.tol,
                cfg.max_iter)
    dt = time.perf_counter() - t0
    return {"value": r.n_iterations / dt, "unit": "matvecs/s", "cores": cores, "kind": "port",
            "sample": f"one relaxed GMRES solve of {cfg.name} ({r.n_iterations} mat-vecs at p "
                      f"{r.orders}, {dt:.1f} s; setup excluded, as the reference's study.py:196-204)",
            "time_to_solution_s": dt}


def run_reference(args, cfg, mesh, world):
    rank, _, _ = dist_env()
    if rank != 0:
        return
    from oracle import fmm_oracle as O
    from paper_1506_05957_b200.configs import CONFIGS  # noqa: F401

    cores = cpu_threads()
    op = O.OracleOperator(mesh, cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
    data = cfg.boundary_data(op.centroids, op.normals)
    x = np.random.default_rng(1).uniform(-1.0, 1.0, op.n)
    # the relaxed schedule the solve follows on this config (pinned by tests/golden/cfg2.npz)
    schedule = [cfg.p_initial, cfg.p_initial, 10, 5] if cfg.name == "cfg2" else [cfg.p_initial]
    del data
    for i in range(args.warmup):
        op.apply(x, schedule[i % len(schedule)])
    t0 = time.perf_counter()
    for i in range(args.steps):
        op.apply(x, schedule[i % len(schedule)])
    dt = time.perf_counter() - t0
    value = args.steps / dt
    line = {
        "metric": f"FMM mat-vecs/s at N={mesh.n_panels} panels (relaxed GMRES, {cfg.name})",
        "value": value, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_desc(cfg, mesh), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "matvecs/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} mat-vecs cycling p over {schedule} (the relaxed "
                                   "schedule); oracle/fmm_oracle.py restates the reference, pinned "
                                   "by tests/golden"},
        "e2e": {"value": value, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU leg
M2L_ROT_MIN_P = 3  # csrc/kernels.cuh: rotation-based M2L from this order up


def m2l_flops(n_pairs, C, p):
    """Algorithmic flops of the M2L formulation the library runs at order p.

    p >= 3, rotation ("point and shoot", m2l_rot.cu): per pair and channel three
    real products on the real and imaginary parts, stage A and C of order
    (n+1) x (n+1) per degree, stage B (p+1-k) x (p+1-k) per order:
    2 flop x 2 parts x (2 S2 + S2), S2 = sum_{i<=p+1} i^2.
    p < 3, dense contraction of half-stored outputs with full inputs:
    8 flop per complex MAC x (p+1)(p+2)/2 x (p+1)^2."""
    if p >= M2L_ROT_MIN_P:
        s2 = (p + 1) * (p + 2) * (2 * p + 3) // 6
        return n_pairs * C * 12.0 * s2
    H = (p + 1) * (p + 2) // 2
    S = (p + 1) ** 2
    return n_pairs * C * H * S * 8.0


def run_ours(args, cfg, mesh, world):
    import torch

    from paper_1506_05957_b200 import _native as N
    from paper_1506_05957_b200.operator import GpuBemOperator
    from paper_1506_05957_b200.solver import RelaxationSchedule, _device_gmres

    rank, _, local = dist_env()
    dist = world > 1
    if dist:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl")
    device = local if dist else 0
    torch.cuda.set_device(device)
    op = GpuBemOperator(mesh, cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu,
                        device=device)
    data = cfg.boundary_data(op.centroids, op.normals)
    b_host = op.assemble_rhs(data)
    if dist:
        from paper_1506_05957_b200.parallel import shard_operator

        shard_operator(op, rank, world)
    n = op.shape[0]
    b_dev = torch.from_numpy(b_host).to(f"cuda:{device}")
    x_dev = torch.empty(n, dtype=torch.float64, device=f"cuda:{device}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{device}")
    sched = RelaxationSchedule(cfg.p_initial, cfg.p_min, cfg.tol, True)
    lib = N.load()
    import ctypes

    res = np.zeros(cfg.max_iter)
    ords = np.zeros(cfg.max_iter, dtype=np.int32)
    nit = ctypes.c_int32(0)
    conv = ctypes.c_int32(0)

    def solve_device():
        N.check(lib.fmmbem_op_gmres_device(op._h, ctypes.c_void_p(b_dev.data_ptr()), cfg.tol,
                                           cfg.p_initial, cfg.p_min, 1, cfg.max_iter,
                                           ctypes.c_void_p(x_dev.data_ptr()), N.dptr(res),
                                           N.i32ptr(ords), ctypes.byref(nit), ctypes.byref(conv)))
        return int(nit.value), [int(o) for o in ords[:nit.value]]

    op.set_timing(False)  # the timed steps run the plain graphs; stages come from a separate pass
    for _ in range(args.warmup):
        flush.zero_()
        torch.cuda.synchronize()
        solve_device()
    op.stage_times(reset=True)
    launches0, applies0, _ = op.counters()
    orders_seen = []
    step_ms = []
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(device) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            k, ords_k = solve_device()
            orders_seen.append(ords_k)
            step_ms.append(op.counters()[2])
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if dist:
            tdist.barrier()
    launches1, applies1, _ = op.counters()
    # per-stage CUDA-event timings: the same solve, instrumented, outside the timed region
    op.set_timing(True)
    solve_device()  # captures the instrumented graphs
    op.stage_times(reset=True)
    for _ in range(max(3, args.steps // 4)):
        flush.zero_()
        torch.cuda.synchronize()
        solve_device()
    stages, calls = op.stage_times(reset=True)
    # the same solve with the near field in line: every kernel has the GPU to itself, so the
    # stage times are the kernels' own durations (the roofline), not their share of a
    # contended step
    op.set_serial(True)
    solve_device()
    op.stage_times(reset=True)
    for _ in range(max(3, args.steps // 4)):
        flush.zero_()
        torch.cuda.synchronize()
        solve_device()
    iso, iso_calls = op.stage_times(reset=True)
    op.set_serial(False)
    op.set_timing(False)
    dev_ms = float(np.sum(step_ms))
    applies = applies1 - applies0
    from paper_1506_05957_b200.parallel import reduce_timing

    # one partitioned job: every rank takes part in the same mat-vecs (strong scaling)
    dev_ms_max, _ = reduce_timing(dev_ms, applies, device=f"cuda:{device}")
    total_applies = float(applies)
    value = total_applies / (dev_ms_max * 1e-3)

    # e2e through the public API: host pinned b -> solve() -> host x
    b_pin = torch.from_numpy(b_host).pin_memory().numpy()
    e2e_ms, e2e_applies, d2h = [], 0, 0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        out = _device_gmres(op, b_pin, sched, cfg.tol, cfg.max_iter)
        e2e_ms.append(1e3 * (time.perf_counter() - t1))
        e2e_applies += out.n_iterations
        m = out.n_iterations
        d2h = 8 * n + 8 + sum(8 * (k + 2) for k in range(m))  # x, ||b||, H columns
    e2e_value = e2e_applies / (np.sum(e2e_ms) * 1e-3)

    # roofline of the dominant kernel (the near field: ~42% of the step in the ncu launch list),
    # from CUDA events on the stream it is launched on
    fp64_peak = N.fp64_peak_tflops(device)
    flat_orders = [p for o in orders_seen for p in o]
    ppf = P2P_FLOPS_PER_INTERACTION[cfg.formulation]
    C = 4 if cfg.formulation == "stokes" else 1
    algo = {"p2p": ppf * op.plan.p2p_interactions * len(flat_orders),
            "m2l": sum(m2l_flops(op.plan.n_m2l, C, p) for p in flat_orders)}
    # per apply: the timed steps' algorithmic work over the instrumented passes' stage times
    algo = {k: v / max(len(flat_orders), 1) for k, v in algo.items()}
    stages = {k: v / max(calls, 1) for k, v in stages.items()}
    iso = {k: v / max(iso_calls, 1) for k, v in iso.items()}
    if iso["p2p"] <= 0.0 or stages["p2p"] <= 0.0:
        raise RuntimeError(f"no stage timings were recorded: {stages} {iso}")
    achieved = algo["p2p"] / (iso["p2p"] * 1e-3) / 1e12
    traffic = None
    tf = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(cfg.name, {}).get("p2p")
    roofline = {
        "kernel": "k_p2p_lapd (near field, double layer)" if cfg.formulation != "stokes"
        else "k_p2p<STOKESLET> (near field)",
        "bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
        "frac": achieved / fp64_peak, "traffic": traffic,
        "timing": "CUDA events around the kernel on its stream; this value from the isolated pass "
                  "(near field in line, the kernel alone on the GPU); in_step = the same kernel "
                  "inside the concurrent step (sharing SMs with the far field)",
        "in_step": {"achieved": algo["p2p"] / (stages["p2p"] * 1e-3) / 1e12,
                    "frac": algo["p2p"] / (stages["p2p"] * 1e-3) / 1e12 / fp64_peak,
                    "ms": stages["p2p"]},
        "peak_source": "live DFMA microkernel on this GPU (MEASURED_PEAKS.json has no fp64 entry)",
        "algorithmic": {
            "p2p": f"{ppf} flop/interaction x {op.plan.p2p_interactions} interactions/apply",
            "m2l": "rotation M2L (p >= 3): 12 flop x sum_{i<=p+1} i^2 per pair and channel; "
                   "p < 3: 8 flop/complex MAC x (p+1)(p+2)/2 x (p+1)^2"},
        "stage_ms_per_apply": stages,
        "stage_ms_per_apply_isolated": iso,
        "stage_share_isolated": {k: v / iso["total"] for k, v in iso.items() if k != "total"},
        "other_kernel": {
            "m2l": {"achieved": algo["m2l"] / (iso["m2l"] * 1e-3) / 1e12,
                    "frac": algo["m2l"] / (iso["m2l"] * 1e-3) / 1e12 / fp64_peak}},
    }
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline_sample(cfg, mesh, b_host)
    line = {
        "metric": f"FMM mat-vecs/s at N={mesh.n_panels} panels (relaxed GMRES, {cfg.name})",
        "value": value, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_desc(cfg, mesh), parallelism=f"shard{world}" if world > 1 else "single"),
        "time_to_solution_ms": dev_ms_max / args.steps,
        "iterations": len(orders_seen[-1]), "orders": orders_seen[-1],
        "wall_s_timed_region": wall,
        "e2e": {"value": e2e_value, "unit": "matvecs/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": d2h, "ms_per_step": float(np.mean(e2e_ms)),
                "api": "paper_1506_05957_b200.solver (fmmbem_op_gmres), host pinned b, host x"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": int(launches1 - launches0),
        "structure": {"p2p_interactions_per_apply": op.plan.p2p_interactions,
                      "m2l_pairs": op.plan.n_m2l, "src_cells": op.plan.n_src_cells,
                      "tgt_cells": op.plan.n_tgt_cells},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    from paper_1506_05957_b200.configs import CONFIGS

    cfg = CONFIGS[args.config]
    mesh = cfg.mesh()
    _, world, _ = dist_env()
    world = max(world, 1)
    if args.impl == "reference":
        run_reference(args, cfg, mesh, world)
    else:
        run_ours(args, cfg, mesh, world)


if __name__ == "__main__":
    main()
