#!/usr/bin/env python
"""Benchmark: FMM mat-vecs/s of relaxed GMRES at N panels on BASELINE.json configs[4] (cfg5).

cfg5 is the largest single-GPU configuration of BASELINE.json (and north_star's strong-scaling
config): icosphere L7, 327 680 panels, Laplace 2nd kind, 8 seeded interior charges, theta 0.5,
n_crit 256, tol 1e-6, p 14 -> 3, unrestarted.  One step = one relaxed-GMRES solve with b
resident in HBM; value = mat-vecs (applies) done / device time, whole job.  ``e2e`` is the same
metric through the public Python API (``solver.solve`` path: host pinned b -> host x).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfgK]

Under torchrun (N > 1) the same solve is partitioned over the N GPUs (strong scaling).
``--impl reference`` times the reference's CPU path on the host cores: the oracle port
(oracle/fmm_oracle.py, pinned to the unmodified reference by tests/golden) with its per-leaf /
per-cell loops spread over every host core (oracle/parallel_oracle.py); one step = one apply,
cycling the relaxed orders the reference's own solve used on this config (tests/golden), rank 0
only.
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

CONFIG_NAME = "cfg5"
P2P_FLOPS_PER_INTERACTION = {"laplace_second": 18, "laplace_first": 11, "stokes": 29}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=CONFIG_NAME)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-leg", action="store_true", help=argparse.SUPPRESS)  # internal subprocess
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload_desc(cfg, mesh, world):
    """The config dict both arms print (the driver compares them)."""
    return {
        "workload": f"{cfg.name}: {mesh.n_panels}-panel {'RBC lattice' if cfg.name == 'cfg4' else 'icosphere'}, "
                    f"{cfg.formulation}, "
                    + (f"{cfg.n_charges} seeded interior charges, " if cfg.n_charges else "")
                    + f"theta {cfg.theta}, n_crit {cfg.n_crit}, relaxed GMRES tol {cfg.tol:g}, "
                    f"p {cfg.p_initial}->{cfg.p_min}, unrestarted",
        "panels": mesh.n_panels,
        "unknowns": mesh.n_panels * (3 if cfg.formulation == "stokes" else 1),
        "gauss_points_far": 4,
        "near_rule": "19-pt degree 9 + 32-node polar singular",
        "step": "one relaxed GMRES solve (b resident in HBM)",
        "l2": "256 MiB buffer written between timed steps (L2 flush)",
        "parallelism": f"shard{world}" if world > 1 else "single",
    }


def golden_orders(cfg):
    """The relaxed orders the UNMODIFIED reference's solve used on this config (tests/golden)."""
    for f in (f"{cfg.name}.npz", f"{cfg.name}_sampled.npz", f"{cfg.name}_solve.npz"):
        path = os.path.join(ROOT, "tests", "golden", f)
        if os.path.exists(path):
            d = np.load(path)
            if "relaxed_orders" in d:
                return [int(v) for v in d["relaxed_orders"]]
    return [cfg.p_initial]


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (NVML, every 10 ms, in a
    thread; the timed region of a cfg5 run is only ~0.2 s)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.sm, self.smax, self.reasons = [], [], set()
        self._stop = None
        self._thr = None
        self.err = None

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            uuid = None
            try:
                import torch

                uuid = str(torch.cuda.get_device_properties(self.gpu).uuid)
            except Exception:
                pass
            h = None
            if uuid:
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hi = pynvml.nvmlDeviceGetHandleByIndex(i)
                    u = pynvml.nvmlDeviceGetUUID(hi)
                    u = u.decode() if isinstance(u, bytes) else u
                    if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                        h = hi
            self.h = h if h is not None else pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nv = pynvml
        except Exception as exc:
            self.err = f"nvml unavailable: {exc}"
            return self
        self._stop = threading.Event()

        def loop():
            nv = self.nv
            while not self._stop.is_set():
                self.sample()
                self._stop.wait(0.01)

        self.sample()
        self._thr = threading.Thread(target=loop, daemon=True)
        self._thr.start()
        return self

    def sample(self):
        nv = self.nv
        try:
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
            self.smax.append(float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for nm, bit in self.REASONS.items():
                if mask & bit:
                    self.reasons.add(nm)
        except Exception as exc:
            self.err = str(exc)

    def __exit__(self, *a):
        if self._thr is not None:
            self._stop.set()
            self._thr.join(timeout=2)
            self.sample()

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"]}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": float(max(self.smax)),
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml 10 ms"}


# ---------------------------------------------------------------- CPU (oracle) legs
def cpu_threads():
    n = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(n)
    except Exception:
        pass
    return n


def host_info():
    """CPU model, core count and the numpy / scipy / BLAS builds the CPU legs run on."""
    info = {"cpu_model": None, "cores": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    import scipy

    info["numpy"] = np.__version__
    info["scipy"] = scipy.__version__
    try:
        from threadpoolctl import threadpool_info

        info["blas"] = [f"{d.get('internal_api')} {d.get('version')} ({d.get('threading_layer')}, "
                        f"{d.get('num_threads')} threads)" for d in threadpool_info()
                        if d.get("user_api") == "blas"]
    except Exception:
        info["blas"] = None
    return info


def oracle_setup(cfg, mesh, orders, workers):
    from oracle import fmm_oracle as O
    from oracle.parallel_oracle import ParallelOracle

    t0 = time.perf_counter()
    op = O.OracleOperator(mesh, cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
    setup_s = time.perf_counter() - t0
    par = ParallelOracle(op, orders, workers=workers)
    return op, par, setup_s


def cpu_leg_main(args, cfg, mesh):
    """Subprocess body of the in-arm cpu_baseline (a fork pool must not inherit a CUDA context):
    one apply at every distinct relaxed order of the reference's solve on this config."""
    cores = cpu_threads()
    orders = golden_orders(cfg)
    op, par, setup_s = oracle_setup(cfg, mesh, orders, cores)
    x = np.random.default_rng(1).uniform(-1.0, 1.0, op.n)
    per_p = {}
    t0 = time.perf_counter()
    for p in sorted(set(orders), reverse=True):
        t1 = time.perf_counter()
        par.apply(x, p)
        per_p[str(p)] = time.perf_counter() - t1
    dt = time.perf_counter() - t0
    par.close()
    # a relaxed solve's mat-vecs at the reference's own orders, from the per-order times
    solve_s = sum(per_p[str(p)] for p in orders)
    print(json.dumps({"value": len(orders) / solve_s, "unit": "matvecs/s", "cores": cores,
                      "kind": "port",
                      "sample": f"one apply of {cfg.name} at each order of the reference's relaxed "
                                f"solve {orders} ({dt:.1f} s of CPU work); value = {len(orders)} "
                                f"mat-vecs / the sum of their apply times. oracle/fmm_oracle.py "
                                "restates the reference (pinned by tests/golden); its leaf/cell "
                                "loops run on every host core (oracle/parallel_oracle.py)",
                      "apply_s_per_p": per_p, "setup_s": setup_s, "host": host_info()}),
          flush=True)


def cpu_baseline_sample(args, cfg):
    """Runs cpu_leg_main in a fresh process (bench.py --cpu-leg) and returns its JSON."""
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-leg", "--config", cfg.name]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=dict(os.environ))
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:  # the GPU line must still print
        return {"value": None, "unit": "matvecs/s", "cores": os.cpu_count(), "kind": "port",
                "sample": f"cpu leg failed: {type(exc).__name__}: {exc}"[:300]}


def run_reference(args, cfg, mesh, world):
    rank, _, _ = dist_env()
    if rank != 0:
        return
    cores = cpu_threads()
    orders = golden_orders(cfg)
    op, par, setup_s = oracle_setup(cfg, mesh, orders, cores)
    x = np.random.default_rng(1).uniform(-1.0, 1.0, op.n)
    for i in range(args.warmup):
        par.apply(x, orders[i % len(orders)])
    t0 = time.perf_counter()
    for i in range(args.steps):
        par.apply(x, orders[i % len(orders)])
    dt = time.perf_counter() - t0
    par.close()
    value = args.steps / dt
    sample = (f"{args.steps} applies of {cfg.name} cycling p over {orders} (the orders of the "
              "reference's own relaxed solve, tests/golden); oracle/fmm_oracle.py restates the "
              "reference (pinned by tests/golden), its leaf/cell loops on all host cores "
              "(oracle/parallel_oracle.py); setup excluded like study.py:196-204")
    line = {
        "metric": f"FMM mat-vecs/s at N={mesh.n_panels} panels (relaxed GMRES, {cfg.name})",
        "value": value, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_desc(cfg, mesh, world), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "matvecs/s", "cores": cores, "kind": "port",
                         "sample": sample, "setup_s": setup_s, "host": host_info()},
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
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    op = GpuBemOperator(mesh, cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu,
                        device=device)
    setup_s = time.perf_counter() - t_setup  # BemOperator.__init__ (bemop.py:50-82), host->host
    data = cfg.boundary_data(op.centroids, op.normals)
    op.assemble_rhs(data)  # first call builds the p=18 tables
    t_rhs = time.perf_counter()
    b_host = op.assemble_rhs(data)
    rhs_s = time.perf_counter() - t_rhs  # assemble_rhs (bemop.py:290-310), host->host
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
                                           cfg.tol, cfg.p_initial, cfg.p_min, 1, cfg.max_iter,
                                           ctypes.c_void_p(x_dev.data_ptr()), N.dptr(res),
                                           N.i32ptr(ords), ctypes.byref(nit), ctypes.byref(conv),
                                           None, None, None))
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
    applies = sum(len(o) for o in orders_seen)  # mat-vecs done by the timed solves
    from paper_1506_05957_b200.parallel import reduce_timing

    # one partitioned job: every rank takes part in the same mat-vecs (strong scaling)
    dev_ms_max, _ = reduce_timing(dev_ms, applies, device=f"cuda:{device}")
    total_applies = float(applies)
    value = total_applies / (dev_ms_max * 1e-3)

    # e2e through the public API: host pinned b -> solve() -> host x
    b_pin = torch.from_numpy(b_host).pin_memory().numpy()
    e2e_ms, e2e_applies, d2h = [], 0, 0
    # warm-up in the timed loop's own pattern: `out` is rebound while the previous result is
    # still alive, so two page-locked result buffers circulate through torch's caching host
    # allocator -- without this the second timed step paid a fresh cudaHostAlloc (3-100 ms)
    out = None
    for _ in range(max(args.warmup, 2)):
        out = _device_gmres(op, b_pin, sched, cfg.tol, cfg.max_iter)
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
                    "frac": algo["m2l"] / (iso["m2l"] * 1e-3) / 1e12 / fp64_peak,
                    "note": "whole M2L stage (rotation kernel + per-target gather of the pair slots), "
                            "averaged over the solve's orders; the rotation kernel alone at p_initial "
                            "is in profiles/ (bound by shared-memory / L1 operand bandwidth)"}},
    }
    # apply(x, p) throughput per order (headline unit): CUDA events around
    # back-to-back device applies on the op's stream, x resident in HBM
    xin = torch.from_numpy(np.random.default_rng(1).uniform(-1.0, 1.0, n)).to(f"cuda:{device}")
    yout = torch.empty_like(xin)
    per_p = {}
    if not dist:
        stream = torch.cuda.current_stream(device)
        for p in sorted(set(p for o in orders_seen for p in o), reverse=True):
            for _ in range(2):
                op.apply_device(xin.data_ptr(), yout.data_ptr(), p, stream=stream.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record(stream)
            for _ in range(reps):
                op.apply_device(xin.data_ptr(), yout.data_ptr(), p, stream=stream.cuda_stream)
            e1.record(stream)
            e1.synchronize()
            per_p[str(p)] = {"applies_per_s": reps / (e0.elapsed_time(e1) * 1e-3),
                             "ms": e0.elapsed_time(e1) / reps}
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline_sample(args, cfg)
    line = {
        "metric": f"FMM mat-vecs/s at N={mesh.n_panels} panels (relaxed GMRES, {cfg.name})",
        "value": value, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_desc(cfg, mesh, world),
        "time_to_solution_ms": dev_ms_max / args.steps,
        "setup_s": setup_s, "rhs_s": rhs_s,
        "apply_per_p": per_p,
        "iterations": len(orders_seen[-1]), "orders": orders_seen[-1],
        "wall_s_timed_region": wall,
        "e2e": {"value": e2e_value, "unit": "matvecs/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": d2h, "ms_per_step": float(np.mean(e2e_ms)),
                "ms_median": float(np.median(e2e_ms)), "ms_max": float(np.max(e2e_ms)),
                "ms_steps": [round(float(v), 3) for v in e2e_ms],
                "api": "paper_1506_05957_b200.solver (fmmbem_op_gmres), host pinned b, host x"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": int(launches1 - launches0),
        "matvecs_timed": applies,
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
    if args.cpu_leg:
        cpu_leg_main(args, cfg, mesh)
    elif args.impl == "reference":
        run_reference(args, cfg, mesh, world)
    else:
        run_ours(args, cfg, mesh, world)


if __name__ == "__main__":
    main()
