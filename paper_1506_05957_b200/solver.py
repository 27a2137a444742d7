"""Relaxed GMRES on the device, with the reference's solver API.

Mirrors ``pkg/src/fmmbem/solver.py``: ``relax_eps`` (20-24), ``schedule_p``
(27-31), ``RelaxationSchedule`` (34-47), ``SolveResult`` (50-66), ``gmres``
(69-134) and ``solve`` (137-143).  The Arnoldi/Givens loop itself runs in
``libfmmbem_b200.so`` (``fmmbem_op_gmres``) with the Krylov basis resident in
HBM; the schedule functions below are the same scalar rules, exposed for
callers and tests.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


def relax_eps(residual, eta):
    """eps_k = min(eta / min(max(r, eta), 1), 1) (solver.py:20-24)."""
    if eta <= 0.0:
        raise ValueError("eta must be positive")
    return min(eta / min(max(residual, eta), 1.0), 1.0)


def schedule_p(residual, eta, p_initial, p_min):
    """p = ceil(-log2 eps) clamped to [p_min, p_initial] (solver.py:27-31)."""
    eps = relax_eps(residual, eta)
    p = math.ceil(-math.log2(eps)) if eps < 1.0 else p_min
    return int(min(p_initial, max(p_min, p)))


@dataclass
class RelaxationSchedule:
    p_initial: int = 12
    p_min: int = 1
    eta: float = 1e-5
    relaxed: bool = True

    def order(self, residual, previous_p):
        if not self.relaxed:
            return self.p_initial
        return min(schedule_p(residual, self.eta, self.p_initial, self.p_min), previous_p)


@dataclass
class SolveResult:
    x: np.ndarray
    residuals: list = field(default_factory=list)
    orders: list = field(default_factory=list)
    converged: bool = False

    @property
    def n_iterations(self):
        return len(self.orders)

    def save_history(self, path):
        """'iteration,residual,p' lines (solver.py:61-66)."""
        with open(path, "w") as fh:
            fh.write("iteration,residual,p\n")
            for k, (r, p) in enumerate(zip(self.residuals, self.orders), start=1):
                fh.write(f"{k},{r:.17g},{p}\n")


def _device_gmres(op, b, schedule, tol, max_iter, callback=None):
    """One fmmbem_op_gmres call: the Arnoldi/Givens loop runs in the library, the
    per-iteration ``callback(k, residual, p)`` is called from inside it (solver.py:122-123)."""
    lib = N.load()
    bb = op._vec(b)
    n = len(bb)
    x = N.host_array(n)
    res = np.zeros(max(max_iter, 1))
    orders = np.zeros(max(max_iter, 1), dtype=np.int32)
    nit = ctypes.c_int32(0)
    conv = ctypes.c_int32(0)
    raised = []
    cb = None
    if callback is not None:
        def _progress(k, r, p, _user):
            try:
                callback(int(k), float(r), int(p))
                return 0
            except BaseException as exc:  # re-raised below, after the library returns
                raised.append(exc)
                return 1

        cb = N.GMRES_CALLBACK(_progress)
    N.check(lib.fmmbem_op_gmres(op._h, N.dptr(bb), float(tol), float(schedule.eta),
                                int(schedule.p_initial), int(schedule.p_min),
                                1 if schedule.relaxed else 0, int(max_iter), N.dptr(x),
                                N.dptr(res), N.i32ptr(orders), ctypes.byref(nit),
                                ctypes.byref(conv), cb, None))
    if raised:
        raise raised[0]
    k = int(nit.value)
    return SolveResult(x=x, residuals=res[:k].tolist(), orders=[int(o) for o in orders[:k]],
                       converged=bool(conv.value))


def _host_gmres(apply_fn, b, schedule, tol, max_iter, callback):
    """The reference loop (solver.py:78-134) around an arbitrary ``apply_fn(x, p)``.

    Only for callables that are not a :class:`GpuBemOperator` apply (a user's own
    operator, a wrapped or preconditioned GPU apply): the mat-vec is whatever the caller
    passes; the MGS / Givens bookkeeping is the reference's, statement for statement."""
    b = np.asarray(b, dtype=float)
    norm_b = np.linalg.norm(b)
    if norm_b == 0.0:
        return SolveResult(x=np.zeros_like(b), converged=True)
    n = len(b)
    basis = [b / norm_b]
    H = np.zeros((max_iter + 1, max_iter))
    cs, sn, g = np.zeros(max_iter), np.zeros(max_iter), np.zeros(max_iter + 1)
    g[0] = norm_b
    result = SolveResult(x=np.zeros(n))
    residual, prev_p = 1.0, schedule.p_initial
    for k in range(max_iter):
        p = schedule.order(residual, prev_p)
        prev_p = p
        w = np.asarray(apply_fn(basis[k], p), dtype=float)
        for j in range(k + 1):
            H[j, k] = basis[j] @ w
            w = w - H[j, k] * basis[j]
        H[k + 1, k] = np.linalg.norm(w)
        basis.append(w / H[k + 1, k] if H[k + 1, k] > 0.0 else np.zeros(n))
        for j in range(k):
            h1 = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
            H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
            H[j, k] = h1
        denom = math.hypot(H[k, k], H[k + 1, k])
        cs[k], sn[k] = H[k, k] / denom, H[k + 1, k] / denom
        H[k, k], H[k + 1, k] = denom, 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        residual = abs(g[k + 1]) / norm_b
        result.residuals.append(residual)
        result.orders.append(p)
        if callback is not None:
            callback(k + 1, residual, p)
        if residual < tol:
            result.converged = True
            break
    m = len(result.orders)
    y = np.linalg.solve(H[:m, :m], g[:m]) if m else np.zeros(0)
    x = np.zeros(n)
    for j in range(m):
        x += y[j] * basis[j]
    result.x = x
    return result


def gmres(apply_fn, b, schedule=None, tol=1e-5, max_iter=100, callback=None):
    """Unrestarted relaxed GMRES (solver.py:69-134).

    With the bound ``apply`` of a :class:`GpuBemOperator` the whole loop runs on the device
    (Krylov basis in HBM, ``fmmbem_op_gmres``); ``schedule.eta`` drives the order and ``tol``
    the stop test, and ``callback(k, residual, p)`` is called after every iteration, as in the
    reference.  Any other callable gets the reference's own host loop around it.
    """
    from .operator import GpuBemOperator

    if schedule is None:
        schedule = RelaxationSchedule(eta=tol, relaxed=False)
    if max_iter < 0:
        raise ValueError("max_iter must be >= 0")
    op = getattr(apply_fn, "__self__", None)
    if isinstance(op, GpuBemOperator) and getattr(apply_fn, "__func__", None) is GpuBemOperator.apply:
        return _device_gmres(op, b, schedule, tol, max_iter, callback)
    return _host_gmres(apply_fn, b, schedule, tol, max_iter, callback)


def solve(operator, b, eta=1e-5, p_initial=12, p_min=1, relaxed=True, max_iter=100,
          callback=None):
    """Relaxed (or fixed-order) GMRES on a device BEM operator (solver.py:137-143)."""
    schedule = RelaxationSchedule(p_initial=p_initial, p_min=p_min, eta=eta, relaxed=relaxed)
    return gmres(operator.apply, b, schedule=schedule, tol=eta, max_iter=max_iter,
                 callback=callback)
