"""Goldens of the reference's study harness (study.py:143-242), run UNMODIFIED here.

Usage: PYTHONPATH=/root/reference/pkg/src:. python tools/make_goldens_study.py
Writes tests/golden/study.npz: run_relaxation_comparison('laplace2', level 3, tol 1e-6,
p 10 -> 3, n_crit (16, 64), repeats 1) and ('stokes', level 2, tol 1e-5, p 12 -> 5,
n_crit (16, 64)) records (iterations, converged, N, n_crit, relaxed; wall times are machine
properties and are not kept) and derived iteration counts / solution difference;
run_convergence('laplace2', levels 1-3, p 10, tol 1e-8, n_crit 32, p_min 3) records
(N, iterations, orders, error) and the derived order.
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from tools.make_goldens import OUT  # noqa: E402

RELAX = [("laplace2", dict(level=3, tol=1e-6, p_initial=10, p_min=3, ncrit_candidates=(16, 64))),
         ("stokes", dict(level=2, tol=1e-5, p_initial=12, p_min=5, ncrit_candidates=(16, 64)))]
CONV = ("laplace2", dict(levels=[1, 2, 3], p=10, tol=1e-8, n_crit=32, p_min=3))


def main():
    from fmmbem import study

    out = {}
    for name, kw in RELAX:
        rep = study.run_relaxation_comparison(name, repeats=1, **kw)
        recs = [{k: r[k] for k in ("N", "n_crit", "relaxed", "iterations", "converged")}
                for r in rep.records]
        out[f"relax_{name}_records"] = np.array(json.dumps(recs))
        out[f"relax_{name}_derived"] = np.array(json.dumps(
            {k: rep.derived[k] for k in ("iterations_relaxed", "iterations_fixed",
                                         "solution_difference")}))
    name, kw = CONV
    rep = study.run_convergence(name, **kw)
    recs = [{k: (list(map(int, r[k])) if k == "orders" else r[k])
             for k in ("N", "iterations", "converged", "orders", "error")} for r in rep.records]
    out["conv_laplace2_records"] = np.array(json.dumps(recs))
    out["conv_laplace2_order"] = np.array(rep.derived["order"])
    np.savez_compressed(os.path.join(OUT, "study.npz"), **out)
    print("wrote study.npz", {k: str(v)[:200] for k, v in out.items()})


if __name__ == "__main__":
    main()
