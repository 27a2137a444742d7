"""Round-2 goldens from the REFERENCE itself (this container only; hours of CPU for cfg4).

Usage: PYTHONPATH=/root/reference/pkg/src:. python tools/make_goldens_r2.py cfg4solve|cfg5p10|cfg2extra ...

  cfg4solve  BASELINE config 4 (64 RBCs, Stokes, 393 216 unknowns): apply(x, 8) on the sampled
             rows, then the relaxed GMRES solve (solver.py:69-134) with max_iter 600 -- orders,
             residuals, the solution on the sampled rows and its norm.  The per-iteration
             history is also streamed to tests/golden/cfg4_solve.progress.txt so a cut run still
             leaves evidence.  Writes tests/golden/cfg4_solve.npz.
  cfg5p10    BASELINE config 5: apply(x, 10) and apply(x, 4) on the sampled rows (the relaxed
             schedule's intermediate orders).  Writes tests/golden/cfg5_mid.npz.
  cfg2extra  BASELINE config 2: full apply(x, p) for p = 5 and 10.  Writes tests/golden/cfg2_mid.npz.

Same input vector and row subset as tools/make_goldens_large.py (x = default_rng(1).uniform(-1,1,n),
rows = sorted default_rng(7).choice(n, 4096)).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from paper_1506_05957_b200.configs import CONFIGS  # noqa: E402
from tools.make_goldens import OUT, mesh_digest  # noqa: E402

N_SAMPLE = 4096


def _op(name):
    import fmmbem
    from fmmbem.bemop import BemOperator

    cfg = CONFIGS[name]
    mesh = cfg.mesh()
    t0 = time.perf_counter()
    op = BemOperator(fmmbem.Mesh(mesh.vertices, mesh.triangles), cfg.formulation, theta=cfg.theta,
                     n_crit=cfg.n_crit, mu=cfg.mu)
    print(f"[{name}] setup {time.perf_counter() - t0:.1f}s", flush=True)
    n = op.shape[0]
    rows = np.sort(np.random.default_rng(7).choice(n, size=min(N_SAMPLE, n), replace=False))
    x = np.random.default_rng(1).uniform(-1.0, 1.0, n)
    return cfg, mesh, op, rows, x


def cfg4solve():
    import fmmbem

    cfg, mesh, op, rows, x = _op("cfg4")
    out = {"mesh_sha256": np.array(mesh_digest(mesh)), "rows": rows}
    t0 = time.perf_counter()
    y = op.apply(x, 8)
    print(f"[cfg4] apply p=8 {time.perf_counter() - t0:.1f}s", flush=True)
    out["apply_p8_rows"] = y[rows]
    out["apply_p8_norm"] = np.array(np.linalg.norm(y))
    path = os.path.join(OUT, "cfg4_solve.npz")
    np.savez_compressed(path, **out)
    b = op.assemble_rhs(cfg.boundary_data(op.centroids, op.normals))
    out["rhs_norm"] = np.array(np.linalg.norm(b))
    prog = open(os.path.join(OUT, "cfg4_solve.progress.txt"), "w")
    t_start = time.perf_counter()

    def cb(k, r, p):
        prog.write(f"{k},{r:.17g},{p},{time.perf_counter() - t_start:.1f}\n")
        prog.flush()

    res = fmmbem.solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min, relaxed=True,
                       max_iter=cfg.max_iter, callback=cb)
    print(f"[cfg4] relaxed solve {time.perf_counter() - t_start:.1f}s iters={len(res.orders)} "
          f"converged={res.converged}", flush=True)
    out["relaxed_orders"] = np.asarray(res.orders, dtype=np.int64)
    out["relaxed_residuals"] = np.asarray(res.residuals)
    out["relaxed_converged"] = np.array(bool(res.converged))
    out["relaxed_x_rows"] = res.x[rows]
    out["relaxed_x_norm"] = np.array(np.linalg.norm(res.x))
    out["relaxed_solve_s"] = np.array(time.perf_counter() - t_start)
    out["drag"] = np.asarray(op.drag_force(res.x))
    np.savez_compressed(path, **out)
    print("[cfg4] wrote", flush=True)


def cfg5p10():
    cfg, mesh, op, rows, x = _op("cfg5")
    out = {"mesh_sha256": np.array(mesh_digest(mesh)), "rows": rows}
    for p in (10, 4):
        t0 = time.perf_counter()
        y = op.apply(x, p)
        print(f"[cfg5] apply p={p} {time.perf_counter() - t0:.1f}s", flush=True)
        out[f"apply_p{p}_rows"] = y[rows]
        out[f"apply_p{p}_norm"] = np.array(np.linalg.norm(y))
        np.savez_compressed(os.path.join(OUT, "cfg5_mid.npz"), **out)
    print("[cfg5] wrote", flush=True)


def cfg2extra():
    cfg, mesh, op, rows, x = _op("cfg2")
    out = {"mesh_sha256": np.array(mesh_digest(mesh))}
    for p in (5, 10):
        out[f"apply_p{p}"] = op.apply(x, p)
    np.savez_compressed(os.path.join(OUT, "cfg2_mid.npz"), **out)
    print("[cfg2] wrote", flush=True)


if __name__ == "__main__":
    for job in sys.argv[1:]:
        globals()[job]()
