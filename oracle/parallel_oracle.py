"""Multi-process form of the oracle's mat-vec, for the CPU timing legs (TEST INFRASTRUCTURE).

``oracle/fmm_oracle.py`` restates the reference's ``BemOperator.apply`` (bemop.py:272-288,
FmmPlan.far_field / near_field, fmm.py:203-419) as single-process numpy loops over leaves,
offsets and cells.  The reference itself runs those loops in one Python thread and only the
zgemm/dgemm inside ``@`` is multi-threaded.  On the GPU box that leaves 15 of 16 host cores
idle, so a baseline timed that way would understate what the CPU path can do.  This module runs
the same per-item arithmetic, item for item, on a fork()ed pool of worker processes (one BLAS
thread each):

  * P2M per source leaf, P2P per target leaf, L2P per target leaf: independent items.
  * M2L per target cell, summing its pairs in the oracle's offset order.
  * M2M / L2L: level-sequential, in the parent process, as in the oracle.

Every output row is written by exactly one worker into shared memory, in the oracle's own
summation order.  Only the BLAS row blocking can differ from the serial oracle, so results
agree to rounding (tests/test_oracle.py checks <= 1e-13 against the serial oracle).  Used only
by ``bench.py`` (``cpu_baseline`` and ``--impl reference``) and the tests; never by the
product path.
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os

import numpy as np

from . import fmm_oracle as O

_CTX = None  # the ParallelOracle the forked workers see


def _shared(shape, dtype):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = mmap.mmap(-1, max(n, 1), flags=mmap.MAP_SHARED | mmap.MAP_ANONYMOUS)
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


def _worker_init():
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass


def _run(task):
    _CTX._task(*task)
    return 0


def _chunks(items, n):
    items = list(items)
    k = max(1, min(len(items), n))
    return [items[i::k] for i in range(k)]  # round robin: leaves differ in size


class ParallelOracle:
    """``apply(x, p)`` of an :class:`oracle.fmm_oracle.OracleOperator` on ``workers`` processes.

    ``orders``: the expansion orders that will be applied (their M2L / M2M / L2L tables are
    built before the pool forks, so the workers share them).
    """

    def __init__(self, op: O.OracleOperator, orders, workers=None):
        self.op = op
        self.plan = op.plan
        self.workers = max(1, int(workers or os.cpu_count() or 1))
        self.orders = sorted(set(int(p) for p in orders))
        pmax = max(self.orders)
        S, T = self.plan.S, self.plan.T
        kind = op.sys_kind
        self.C = {"laplace_single": 1, "laplace_double": 1, "stokeslet": 4, "stresslet": 7}[kind]
        self.grad = kind in ("stokeslet", "stresslet")
        ns, nt, C = len(S.points), len(T.points), self.C
        self.q = _shared((C, ns), np.float64)
        self.d = _shared((C, ns, 3), np.float64)
        self.M = _shared((len(S.center) * C * O.nco(pmax),), np.complex128)
        self.L = _shared((len(T.center) * C * O.nco(pmax),), np.complex128)
        self.pot = _shared((2, C, nt), np.float64)       # far, near
        self.gr = _shared((2, C, nt, 3), np.float64)
        # M2L pairs grouped per target cell in the oracle's offset order (fmm.py:292-314)
        pairs = self.plan.m2l_pairs
        self.m2l = {}
        if len(pairs):
            Dq = T.center[pairs[:, 1]] - S.center[pairs[:, 0]]
            quantum = self.plan.root_half * 2.0 ** -22
            keys = np.round(Dq / quantum).astype(np.int64)
            self.uk, inv = np.unique(keys, axis=0, return_inverse=True)
            inv = inv.ravel()
            order = np.lexsort((np.arange(len(inv)), inv))  # by offset, then pair index
            by_t = {}
            for i in order:
                by_t.setdefault(int(pairs[i, 1]), []).append(i)
            self.m2l_tgt = by_t
            self.m2l_inv = inv
            for p in self.orders:
                if p not in self.plan._igrid:
                    self.plan._igrid[p] = O.solid_harmonics(self.uk * quantum, 2 * p, irregular=True)
                g, sg = O._m2l_gather(p)
                self.m2l[p] = (g, sg)
        for p in self.orders:
            self.plan._operators(S, p, "m2m")
            self.plan._operators(T, p, "l2l")
        self.near_items = sorted(self.plan.near.items())
        self.src_leaves = list(S.leaves)
        self.tgt_leaves = list(T.leaves)
        self.m2l_cells = sorted(self.m2l_tgt) if len(pairs) else []
        global _CTX
        _CTX = self
        self.pool = mp.get_context("fork").Pool(self.workers, initializer=_worker_init)

    def close(self):
        if self.pool is not None:
            self.pool.terminate()
            self.pool = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ worker side
    def _Mv(self, p):
        S = self.plan.S
        return self.M[:len(S.center) * self.C * O.nco(p)].reshape(len(S.center), self.C, O.nco(p))

    def _Lv(self, p):
        T = self.plan.T
        return self.L[:len(T.center) * self.C * O.nco(p)].reshape(len(T.center), self.C, O.nco(p))

    def _task(self, what, chunk, p, has_q, has_d):
        S, T = self.plan.S, self.plan.T
        q = self.q if has_q else None
        d = self.d if has_d else None
        bodies = self.plan._bodies
        if what == "p2m":                       # fmm.py:235-259
            M = self._Mv(p)
            for leaf in chunk:
                b = bodies(S, leaf)
                R = O.solid_harmonics(S.points[b] - S.center[leaf], p)
                acc = np.zeros((self.C, O.nco(p)), dtype=complex)
                if q is not None:
                    acc += q[:, b] @ R
                if d is not None:
                    gx, gy, gz = O.regular_grad(R, p)
                    acc += d[:, b, 0] @ gx + d[:, b, 1] @ gy + d[:, b, 2] @ gz
                M[leaf] = acc
        elif what == "m2l":                     # fmm.py:292-314
            M, L = self._Mv(p), self._Lv(p)
            g, sg = self.m2l[p]
            Ig = self.plan._igrid[p]
            pairs = self.plan.m2l_pairs
            for t in chunk:
                acc = np.zeros((self.C, O.nco(p)), dtype=complex)
                for i in self.m2l_tgt[t]:
                    Tm = sg[:, None] * np.conj(Ig[self.m2l_inv[i]][g])
                    acc += M[pairs[i, 0]] @ Tm.T
                L[t] = acc
        elif what == "l2p":                     # fmm.py:319-336
            L = self._Lv(p)
            for leaf in chunk:
                b = bodies(T, leaf)
                R = O.solid_harmonics(T.points[b] - T.center[leaf], p)
                self.pot[0][:, b] = np.real(L[leaf] @ R.T)
                if self.grad:
                    for k, gk in enumerate(O.regular_grad(R, p)):
                        self.gr[0][:, b, k] = np.real(L[leaf] @ gk.T)
        elif what == "p2p":                     # fmm.py:356-419
            for t, srcs in chunk:
                ti = bodies(T, t)
                si = np.sort(np.concatenate([bodies(S, s) for s in srcs]))
                r = T.points[ti][:, None, :] - S.points[si][None, :, :]
                r2 = np.einsum("abk,abk->ab", r, r)
                inv = np.where(r2 > 0.0, 1.0 / np.sqrt(np.where(r2 > 0.0, r2, 1.0)), 0.0)
                i3 = inv ** 3
                pot = np.zeros((self.C, len(ti)))
                grad = np.zeros((self.C, len(ti), 3)) if self.grad else None
                if q is not None:
                    pot += q[:, si] @ inv.T
                    if self.grad:
                        grad -= np.einsum("cs,tsk,ts->ctk", q[:, si], r, i3)
                if d is not None:
                    rd = np.einsum("tsk,csk->cts", r, d[:, si])
                    pot += np.einsum("cts,ts->ct", rd, i3)
                    if self.grad:
                        grad += np.einsum("csk,ts->ctk", d[:, si], i3)
                        grad -= 3.0 * np.einsum("cts,tsk,ts->ctk", rd, r, i3 * inv * inv)
                self.pot[1][:, ti] = pot
                if self.grad:
                    self.gr[1][:, ti] = grad

    def _map(self, what, items, p, has_q, has_d):
        tasks = [(what, ch, p, has_q, has_d) for ch in _chunks(items, 4 * self.workers)]
        self.pool.map(_run, tasks, chunksize=1)

    # ------------------------------------------------------------ parent side
    def _fields(self, q, d, p):
        """far_field + near_field (pot, grad) of the oracle plan, in parallel."""
        S, T = self.plan.S, self.plan.T
        has_q, has_d = q is not None, d is not None
        if has_q:
            self.q[:] = q
        if has_d:
            self.d[:] = d
        self.pot[:] = 0.0
        if self.grad:
            self.gr[:] = 0.0
        # P2M and the near field only need the densities
        self._map("p2p", self.near_items, p, has_q, has_d)
        self._map("p2m", self.src_leaves, p, has_q, has_d)
        M = self._Mv(p)
        nonleaf = np.array([len(k) > 0 for k in S.children])
        M[nonleaf] = 0.0
        up = self.plan._operators(S, p, "m2m")
        for lev in range(int(S.level.max()), 0, -1):          # fmm.py:268-290 (oracle order)
            for c in np.flatnonzero(S.level == lev):
                dd = S.center[c] - S.center[S.parent[c]]
                Tm = up[(lev, tuple(np.sign(dd).astype(int)))]
                M[S.parent[c]] += M[c] @ Tm.T
        L = self._Lv(p)
        L[:] = 0.0
        self._map("m2l", self.m2l_cells, p, has_q, has_d)
        down = self.plan._operators(T, p, "l2l")
        for lev in range(1, int(T.level.max()) + 1):
            for c in np.flatnonzero(T.level == lev):
                dd = T.center[c] - T.center[T.parent[c]]
                Tm = down[(lev, tuple(np.sign(dd).astype(int)))]
                L[c] += L[T.parent[c]] @ Tm.T
        self._map("l2p", self.tgt_leaves, p, has_q, has_d)
        pot = self.pot[0] + self.pot[1]
        grad = (self.gr[0] + self.gr[1]) if self.grad else None
        return pot, grad

    def apply(self, x, p=12):
        """OracleOperator.apply (bemop.py:272-288) with the plan's loops on the pool."""
        op = self.op
        if p not in self.orders:
            raise ValueError(f"order {p} was not prepared (orders={self.orders})")
        x = np.asarray(x, float)
        kind = op.sys_kind
        if kind in ("laplace_single", "laplace_double"):
            s = op.src_weight * x[op.src_panel]
            if kind == "laplace_single":
                pot, _ = self._fields(s[None], None, p)
            else:
                pot, _ = self._fields(None, (s[:, None] * op.src_normal)[None], p)
            out = pot[0] / O.FOUR_PI + op.c_sys @ x
            return 0.5 * x - out if op.formulation == "laplace_second" else out
        f = op.src_weight[:, None] * x.reshape(op.P, 3)[op.src_panel]
        q = np.vstack([f.T, np.einsum("si,si->s", op.src_pos, f)])   # fmm.py:422-425
        pot, grad = self._fields(q, None, p)
        u = pot[:3].T - np.einsum("tc,cti->ti", op.centroids, grad[:3]) + grad[3]
        return (u.reshape(-1) + op.c_sys @ x) / (O.EIGHT_PI * op.mu)
