"""Run BASELINE.json's five configurations end to end on the GPU.

python tools/run_configs.py [cfg1 cfg2 ...] > out.jsonl

Per config: device setup (plan + corrections), RHS assembly, relaxed (and for
cfg2 also fixed-p) GMRES with the device solver, time-to-solution (GMRES loop
only, CUDA events), iterations / p history, accuracy vs the exact potential
(Laplace) or the Stokes drag 6 pi mu U a (sphere), and per-stage apply times.
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from paper_1506_05957_b200.configs import CONFIGS  # noqa: E402
from paper_1506_05957_b200.operator import GpuBemOperator  # noqa: E402
from paper_1506_05957_b200.solver import solve  # noqa: E402


def run(name):
    cfg = CONFIGS[name]
    t0 = time.perf_counter()
    mesh = cfg.mesh()
    t_mesh = time.perf_counter() - t0
    t0 = time.perf_counter()
    op = GpuBemOperator(mesh, cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
    t_setup = time.perf_counter() - t0
    data = cfg.boundary_data(op.centroids, op.normals)
    t0 = time.perf_counter()
    b = op.assemble_rhs(data)
    t_rhs = time.perf_counter() - t0
    out = {"config": name, "panels": mesh.n_panels, "unknowns": op.shape[0], "mesh_s": t_mesh,
           "setup_s": t_setup, "rhs_s": t_rhs, "p2p_interactions": op.plan.p2p_interactions,
           "m2l_pairs": op.plan.n_m2l}
    for relaxed in ((True, False) if name == "cfg2" else (True,)):
        solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min, relaxed=relaxed,
              max_iter=cfg.max_iter)  # warm: graphs per p
        # time to solution: the plain graphs (CUDA events around the device GMRES call)
        res = solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min, relaxed=relaxed,
                    max_iter=cfg.max_iter)
        ms = op.counters()[2]
        # per-stage times from a separate instrumented solve
        op.set_timing(True)
        solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min, relaxed=relaxed,
              max_iter=cfg.max_iter)  # (captures the instrumented graphs)
        op.stage_times(reset=True)
        solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min, relaxed=relaxed,
              max_iter=cfg.max_iter)
        st, calls = op.stage_times(reset=True)
        op.set_timing(False)
        tag = "relaxed" if relaxed else "fixed"
        rec = {"iterations": res.n_iterations, "orders": res.orders, "converged": res.converged,
               "time_to_solution_ms": ms, "final_residual": res.residuals[-1] if res.residuals else None,
               "stage_ms_per_apply": {k: v / max(calls, 1) for k, v in st.items()}}
        ex = cfg.exact_potential(op.centroids)
        if ex is not None:
            rec["err_vs_exact"] = float(np.linalg.norm(res.x - ex) / np.linalg.norm(ex))
        if cfg.formulation == "stokes":
            rec["drag"] = op.drag_force(res.x).tolist()
            if cfg.extra.get("flow", "uniform") == "uniform":
                rec["drag_rel_err"] = abs(rec["drag"][0] - 6 * np.pi * cfg.mu) / (6 * np.pi * cfg.mu)
        out[tag] = rec
    return out


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]:
        print(json.dumps(run(nm)), flush=True)
