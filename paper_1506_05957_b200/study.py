"""Relaxed-vs-fixed comparison with per-variant n_crit sweeps, on the device path.

SURVEY.md §8(f) item 3.  Mirrors the reference's study harness
(`study.py:207-242` run_relaxation_comparison, `:143-191` run_convergence,
`:21-40` observed_order / richardson, `:43-92` StudyReport) with
GpuBemOperator + the device GMRES in place of BemOperator + numpy.  The
paper's "bloated far field" tuning (`PAPER.md:331`) changes on a B200, where
the near field is the cheap part: relaxation only shortens the far field, so
each variant keeps its own fastest n_crit.

Timing is wall clock around `solve()` (host data in, host solution out), the
way the reference times it; the device work inside is synchronous.
"""

from __future__ import annotations

import json
import time

import numpy as np

from .fmm import KernelKind, evaluate
from .meshes import make_octasphere, make_rbc
from .operator import Formulation, GpuBemOperator, GpuFmmPlan
from .solver import solve

__all__ = ["StudyReport", "observed_order", "richardson", "run_relaxation_comparison",
           "run_convergence", "run_scaling"]


def observed_order(f1, f2, f3, c=4.0):
    """ln((f2 - f1) / (f3 - f2)) / ln(c) for a refinement triple (factor c > 1)."""
    if c <= 1.0:
        raise ValueError("refinement ratio c must exceed 1")
    ratio_den = f3 - f2
    if ratio_den == 0.0 or (f2 - f1) / ratio_den <= 0.0:
        raise ValueError("triple is not monotone; order undefined")
    return float(np.log((f2 - f1) / ratio_den) / np.log(c))


def richardson(f1, f2, f3):
    """Aitken/Richardson limit (f1 f3 - f2^2) / (f1 - 2 f2 + f3) of a triple."""
    d = f1 - 2.0 * f2 + f3
    if d == 0.0:
        raise ValueError("degenerate triple; extrapolation undefined")
    return float((f1 * f3 - f2 * f2) / d)


class StudyReport:
    """Records (one dict per solve) + parameters + derived values.

    Same on-disk format as the reference's report: one `key = <json>` line per
    item (`kind`, `param.*`, `record.<i>`, `derived.*`), plus a CSV view.
    """

    def __init__(self, kind, params=None, records=None, derived=None):
        self.kind = kind
        self.params = dict(params or {})
        self.records = list(records or [])
        self.derived = dict(derived or {})

    def _lines(self):
        yield "kind", self.kind
        for k, v in self.params.items():
            yield f"param.{k}", v
        for i, r in enumerate(self.records):
            yield f"record.{i}", r
        for k, v in self.derived.items():
            yield f"derived.{k}", v

    def write(self, path):
        with open(path, "w") as fh:
            for key, val in self._lines():
                fh.write(f"{key} = {json.dumps(val)}\n")

    @classmethod
    def read(cls, path):
        out = cls("")
        recs = {}
        with open(path) as fh:
            for line in fh:
                key, sep, raw = line.rstrip("\n").partition(" = ")
                if not sep:
                    continue
                val = json.loads(raw)
                head, _, tail = key.partition(".")
                if key == "kind":
                    out.kind = val
                elif head == "param":
                    out.params[tail] = val
                elif head == "record":
                    recs[int(tail)] = val
                elif head == "derived":
                    out.derived[tail] = val
        out.records = [recs[i] for i in sorted(recs)]
        return out

    def write_csv(self, path):
        cols = list(dict.fromkeys(k for r in self.records for k in r))
        with open(path, "w") as fh:
            fh.write(",".join(cols) + "\n")
            for r in self.records:
                fh.write(",".join(json.dumps(r.get(c, "")) for c in cols) + "\n")


_PROBLEMS = {"laplace1": Formulation.LAPLACE_FIRST, "laplace2": Formulation.LAPLACE_SECOND,
             "stokes": Formulation.STOKES}


def sphere_problem(problem, level, theta, n_crit, mu=1e-3):
    """(operator, boundary data, exact per-panel solution or None) on the unit sphere
    (octahedron refinement, 8·4^level panels; reference `study.py:102-117`).

    laplace1: phi = 1 given, exact q = 1; laplace2: q = 1 given, exact phi = 1;
    stokes: ambient velocity (1, 0, 0), exact drag 6 pi mu."""
    if problem not in _PROBLEMS:
        raise ValueError(f"unknown problem {problem!r}")
    mesh = make_octasphere(level)
    op = GpuBemOperator(mesh, _PROBLEMS[problem], theta=theta, n_crit=n_crit, mu=mu)
    if problem == "stokes":
        return op, np.tile([1.0, 0.0, 0.0], (mesh.n_panels, 1)), None
    return op, np.ones(mesh.n_panels), np.ones(mesh.n_panels)


def solution_error(op, problem, x, exact):
    """Area-weighted relative L2 error, or the relative drag error for Stokes."""
    if problem == "stokes":
        ref = 6.0 * np.pi * op.mu
        return float(abs(op.drag_force(x)[0] - ref) / ref)
    w = np.asarray(op.areas)
    return float(np.sqrt(w @ (x - exact) ** 2 / (w @ exact ** 2)))


def _timed(op, b, repeats, warmup=1, **kw):
    for _ in range(max(0, warmup)):  # first use of an order instantiates its CUDA graph
        solve(op, b, **kw)
    times, res = [], None
    for _ in range(max(1, repeats)):
        t0 = time.perf_counter()
        res = solve(op, b, **kw)
        times.append(time.perf_counter() - t0)
    return res, float(np.mean(times)), float(np.min(times)), float(np.max(times))


def run_relaxation_comparison(problem, level, tol=1e-5, p_initial=12, p_min=1, theta=0.5,
                              ncrit_candidates=(126,), mu=1e-3, repeats=3, max_iter=100,
                              warmup=1):
    """Relaxed and fixed-order solves for every candidate n_crit; each variant keeps its
    fastest n_crit.  `warmup` untimed solves per variant come first (instantiating an
    order's CUDA graph is setup, like the reference's per-p operator cache).  derived:
    speedup = best fixed time / best relaxed time, the two iteration counts, and the
    relative difference of the two solutions."""
    rep = StudyReport("relaxation", dict(problem=problem, level=level, tol=tol,
                                         p_initial=p_initial, p_min=p_min, theta=theta,
                                         repeats=repeats, warmup=warmup,
                                         ncrit_candidates=list(ncrit_candidates)))
    best, xbest = {}, {}
    for n_crit in ncrit_candidates:
        op, data, _ = sphere_problem(problem, level, theta, n_crit, mu)
        try:
            b = op.assemble_rhs(data)
            for relaxed in (True, False):
                res, t, tmin, tmax = _timed(op, b, repeats, warmup, eta=tol, p_initial=p_initial,
                                            p_min=p_min if relaxed else p_initial,
                                            relaxed=relaxed, max_iter=max_iter)
                rec = dict(N=op.n_panels, n_crit=n_crit, relaxed=relaxed,
                           iterations=res.n_iterations, converged=res.converged,
                           time=t, time_min=tmin, time_max=tmax)
                rep.records.append(rec)
                if relaxed not in best or t < best[relaxed]["time"]:
                    best[relaxed], xbest[relaxed] = rec, np.array(res.x)
        finally:
            op.close()
    rep.derived["speedup"] = best[False]["time"] / best[True]["time"]
    rep.derived["best_ncrit_relaxed"] = best[True]["n_crit"]
    rep.derived["best_ncrit_fixed"] = best[False]["n_crit"]
    rep.derived["iterations_relaxed"] = best[True]["iterations"]
    rep.derived["iterations_fixed"] = best[False]["iterations"]
    rep.derived["solution_difference"] = float(
        np.linalg.norm(xbest[True] - xbest[False]) / np.linalg.norm(xbest[False]))
    return rep


def run_convergence(problem, levels, p=12, tol=1e-6, theta=0.5, n_crit=126, p_min=1,
                    relaxed=True, mu=1e-3, max_iter=100):
    """Solution error (or drag) over a refinement sequence and the observed order
    (reference `study.py:143-191`); "rbc" solves the red-blood-cell drag problem."""
    levels = list(levels)
    if len(levels) < 3:
        raise ValueError("need at least 3 mesh levels")
    rep = StudyReport("convergence", dict(problem=problem, p=p, tol=tol, theta=theta,
                                          n_crit=n_crit, p_min=p_min, relaxed=relaxed))
    vals, counts = [], []
    for level in levels:
        if problem == "rbc":
            mesh = make_rbc(level)
            op = GpuBemOperator(mesh, Formulation.STOKES, theta=theta, n_crit=n_crit, mu=mu)
            data, exact = np.tile([1.0, 0.0, 0.0], (mesh.n_panels, 1)), None
        else:
            op, data, exact = sphere_problem(problem, level, theta, n_crit, mu)
        try:
            b = op.assemble_rhs(data)
            t0 = time.perf_counter()
            res = solve(op, b, eta=tol, p_initial=p, p_min=p_min, relaxed=relaxed,
                        max_iter=max_iter)
            rec = dict(N=op.n_panels, iterations=res.n_iterations, converged=res.converged,
                       time=time.perf_counter() - t0, orders=list(map(int, res.orders)))
            if problem in ("stokes", "rbc"):
                rec["drag"] = float(op.drag_force(res.x)[0])
            rec_val = rec["drag"] if problem == "rbc" else solution_error(op, problem, res.x, exact)
            if problem != "rbc":
                rec["error"] = rec_val
        finally:
            op.close()
        vals.append(rec_val)
        counts.append(rec["N"])
        rep.records.append(rec)
    if problem == "rbc":
        f1, f2, f3 = vals[-3:]
        rep.derived["extrapolated_drag"] = richardson(f1, f2, f3)
        rep.derived["order"] = observed_order(f1, f2, f3, c=counts[-1] / counts[-2])
    else:
        idx = range(1, len(vals) - 1) if len(vals) >= 5 else [len(vals) // 2]
        orders = []
        for i in idx:
            try:
                orders.append(observed_order(vals[i - 1], vals[i], vals[i + 1],
                                             c=counts[i] / counts[i - 1]))
            except ValueError:
                pass
        rep.derived["orders"] = orders
        rep.derived["order"] = float(np.mean(orders)) if orders else float("nan")
    return rep


def run_scaling(sizes, p=5, n_crit=126, theta=0.5, repeats=1, seed=0, warmup=1):
    """Wall time of one Laplace single-layer tree evaluation (far + near field, plan
    prebuilt) over problem sizes, uniform random points in the unit cube, and the
    fitted log-log slope (reference `study.py:245-273`; ~1 for linear scaling)."""
    sizes = [int(n) for n in sizes]
    rng = np.random.default_rng(seed)
    rep = StudyReport("scaling", dict(p=p, n_crit=n_crit, theta=theta, repeats=repeats, seed=seed))
    times = []
    for n in sizes:
        pos = rng.uniform(0.0, 1.0, size=(n, 3))
        q = rng.uniform(-1.0, 1.0, size=n)
        plan = GpuFmmPlan(pos, pos, n_crit=n_crit, theta=theta)
        try:
            for _ in range(max(0, warmup)):
                evaluate(KernelKind.LAPLACE_SINGLE, pos, q, pos, p=p, plan=plan)
            ts = []
            for _ in range(max(1, repeats)):
                t0 = time.perf_counter()
                evaluate(KernelKind.LAPLACE_SINGLE, pos, q, pos, p=p, plan=plan)
                ts.append(time.perf_counter() - t0)
        finally:
            plan.close()
        times.append(float(np.mean(ts)))
        rep.records.append(dict(N=n, time=times[-1], time_min=float(min(ts)), time_max=float(max(ts))))
    if len(sizes) >= 2:
        rep.derived["slope"] = float(np.polyfit(np.log(sizes), np.log(times), 1)[0])
    return rep
