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


def _device_gmres(op, b, schedule, tol, max_iter):
    lib = N.load()
    bb = op._vec(b)
    n = len(bb)
    x = np.empty(n)
    res = np.zeros(max(max_iter, 1))
    orders = np.zeros(max(max_iter, 1), dtype=np.int32)
    nit = ctypes.c_int32(0)
    conv = ctypes.c_int32(0)
    N.check(lib.fmmbem_op_gmres(op._h, N.dptr(bb), float(tol), int(schedule.p_initial),
                                int(schedule.p_min), 1 if schedule.relaxed else 0, int(max_iter),
                                N.dptr(x), N.dptr(res), N.i32ptr(orders), ctypes.byref(nit),
                                ctypes.byref(conv)))
    k = int(nit.value)
    return SolveResult(x=x, residuals=res[:k].tolist(), orders=[int(o) for o in orders[:k]],
                       converged=bool(conv.value))


def gmres(apply_fn, b, schedule=None, tol=1e-5, max_iter=100, callback=None):
    """Unrestarted relaxed GMRES (solver.py:69-134) on a device operator.

    ``apply_fn`` must be the bound ``apply`` of a :class:`GpuBemOperator`
    (the whole loop then runs on the device).  For an arbitrary Python
    callable use the reference's own ``fmmbem.solver.gmres``; a
    ``GpuBemOperator.apply`` plugs into it unchanged.
    """
    from .operator import GpuBemOperator

    op = getattr(apply_fn, "__self__", None)
    if not isinstance(op, GpuBemOperator):
        raise TypeError("gmres() runs on the device: pass GpuBemOperator.apply "
                        "(use fmmbem.solver.gmres for host callables)")
    if schedule is None:
        schedule = RelaxationSchedule(eta=tol, relaxed=False)
    if max_iter < 0:
        raise ValueError("max_iter must be >= 0")
    out = _device_gmres(op, b, schedule, tol, max_iter)
    if callback is not None:
        for k, (r, p) in enumerate(zip(out.residuals, out.orders), start=1):
            callback(k, r, p)
    return out


def solve(operator, b, eta=1e-5, p_initial=12, p_min=1, relaxed=True, max_iter=100,
          callback=None):
    """Relaxed (or fixed-order) GMRES on a device BEM operator (solver.py:137-143)."""
    schedule = RelaxationSchedule(p_initial=p_initial, p_min=p_min, eta=eta, relaxed=relaxed)
    return gmres(operator.apply, b, schedule=schedule, tol=eta, max_iter=max_iter,
                 callback=callback)
