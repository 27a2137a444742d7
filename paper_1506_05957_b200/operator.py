"""Drop-in device replacements for ``BemOperator`` and ``FmmPlan``.

``GpuBemOperator`` has the constructor, methods and attributes of the
reference ``fmmbem.bemop.BemOperator`` (``pkg/src/fmmbem/bemop.py:43-315``),
so ``fmmbem.solver.solve(op, b, ...)`` / ``gmres(op.apply, ...)`` run
unchanged on top of it, and ``paper_1506_05957_b200.solver.solve`` runs the
whole relaxed GMRES on the device.  ``GpuFmmPlan`` mirrors ``FmmPlan``
(``fmm.py:128-419``) for the N-body far/near field API.

Host work here is limited to the O(P) panel geometry (bit-identical to
``quadrature.py:86-121``, see ``geometry.py``) and argument plumbing; the
octree, traversal, correction assembly and every mat-vec run in
``libfmmbem_b200.so``.
"""

from __future__ import annotations

import ctypes
import enum

import numpy as np

from . import _native as N
from .geometry import PanelSet, gauss_legendre

FOUR_PI = 4.0 * np.pi
EIGHT_PI = 8.0 * np.pi


class Formulation(enum.Enum):
    """Same values as the reference enum (bemop.py:33-40)."""

    LAPLACE_FIRST = "laplace_first"
    LAPLACE_SECOND = "laplace_second"
    STOKES = "stokes"


_FORM_CODE = {Formulation.LAPLACE_FIRST: 0, Formulation.LAPLACE_SECOND: 1, Formulation.STOKES: 2}


def _formulation(f) -> Formulation:
    if isinstance(f, Formulation):
        return f
    return Formulation(getattr(f, "value", f))


class GpuFmmPlan:
    """Trees + traversal on the device (``FmmPlan.__init__``, fmm.py:131-168).

    Only ``policy="fmm"`` is served (the hot path); the reference's treecode
    policy (M2P) is outside this build's scope.
    """

    def __init__(self, src_pos, tgt_pos, n_crit=126, theta=0.5, policy="fmm", max_depth=20,
                 device=0, _handle=None, _owner=None):
        if policy != "fmm":
            raise NotImplementedError("only policy='fmm' is implemented on the device")
        self._lib = N.load()
        self.policy = policy
        self.theta = theta
        self.device = device
        self._owner = _owner
        if _handle is not None:
            self._h = _handle
            self._owned = False
        else:
            src = N.f64(np.atleast_2d(src_pos))
            tgt = N.f64(np.atleast_2d(tgt_pos))
            if src.ndim != 2 or src.shape[1] != 3 or len(src) == 0 or tgt.ndim != 2 \
                    or tgt.shape[1] != 3 or len(tgt) == 0:
                raise ValueError("points must be a nonempty (N, 3) array")
            if not 0.0 < theta < 1.0:
                raise ValueError("theta must be in (0, 1)")
            if n_crit < 1:
                raise ValueError("n_crit must be >= 1")
            h = ctypes.c_void_p()
            N.check(self._lib.fmmbem_plan_create(N.dptr(src), len(src), N.dptr(tgt), len(tgt),
                                                 int(n_crit), float(theta), int(max_depth),
                                                 int(device), ctypes.byref(h)))
            self._h = h
            self._owned = True
        s = np.zeros(10, dtype=np.int64)
        N.check(self._lib.fmmbem_plan_sizes(self._h, N.i64ptr(s)))
        (self.n_src_cells, self.n_tgt_cells, self.n_src_leaves, self.n_tgt_leaves, self.n_m2l,
         self.n_p2p, self.n_src_levels, self.n_tgt_levels, self.p2p_interactions,
         self.n_m2l_offsets) = (int(v) for v in s)
        self._ns = None
        self._nt = None

    def close(self):
        if getattr(self, "_owned", False) and self._h:
            self._lib.fmmbem_plan_destroy(self._h)
            self._h = None
            self._owned = False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- structure (compare with the reference by content) ---------------------
    def tree(self, which: str = "src") -> dict:
        w = 0 if which == "src" else 1
        nc = self.n_src_cells if w == 0 else self.n_tgt_cells
        npts = self._npoints(w)
        out = dict(perm=np.empty(npts, np.int64), center=np.empty((nc, 3)), half_width=np.empty(nc),
                   level=np.empty(nc, np.int32), parent=np.empty(nc, np.int32),
                   body_start=np.empty(nc, np.int64), body_count=np.empty(nc, np.int64),
                   is_leaf=np.empty(nc, np.uint8))
        N.check(self._lib.fmmbem_plan_tree(
            self._h, w, N.i64ptr(out["perm"]), N.dptr(out["center"]), N.dptr(out["half_width"]),
            N.i32ptr(out["level"]), N.i32ptr(out["parent"]), N.i64ptr(out["body_start"]),
            N.i64ptr(out["body_count"]), N.u8ptr(out["is_leaf"])))
        out["is_leaf"] = out["is_leaf"].astype(bool)
        return out

    def _npoints(self, w):
        if w == 0:
            if self._ns is None:
                self._ns = int(self._count_points(0))
            return self._ns
        if self._nt is None:
            self._nt = int(self._count_points(1))
        return self._nt

    def _count_points(self, w):
        nc = self.n_src_cells if w == 0 else self.n_tgt_cells
        cnt = np.empty(nc, np.int64)
        N.check(self._lib.fmmbem_plan_tree(self._h, w, None, None, None, None, None, None,
                                           N.i64ptr(cnt), None))
        return cnt[0]  # the root holds every body

    def pairs(self, which: str) -> np.ndarray:
        w = 0 if which == "m2l" else 1
        n = self.n_m2l if w == 0 else self.n_p2p
        out = np.empty((n, 2), np.int32)
        if n:
            N.check(self._lib.fmmbem_plan_pairs(self._h, w, N.i32ptr(out)))
        return out.astype(np.intp)

    @property
    def m2l_pairs(self):
        return self.pairs("m2l")

    @property
    def p2p_pairs(self):
        return self.pairs("p2p")

    def interaction_counts(self) -> np.ndarray:
        """Sources accounted per target via the pair lists (fmm.py:182-191)."""
        st, tt = self.tree("src"), self.tree("tgt")
        counts = np.zeros(len(tt["perm"]))
        for pairs in (self.m2l_pairs, self.p2p_pairs):
            if len(pairs) == 0:
                continue
            add = np.zeros(len(tt["body_count"]))
            np.add.at(add, pairs[:, 1], st["body_count"][pairs[:, 0]])
            for c in np.flatnonzero(add):
                s = tt["body_start"][c]
                counts[tt["perm"][s:s + tt["body_count"][c]]] += add[c]
        return counts

    # -- evaluation ---------------------------------------------------------------
    def _evaluate(self, charges, dipoles, p, want_gradient, parts):
        single = (charges is not None and np.asarray(charges).ndim == 1) or (
            charges is None and np.asarray(dipoles).ndim == 2)
        q = None if charges is None else N.f64(np.atleast_2d(charges))
        d = None
        if dipoles is not None:
            d = N.f64(dipoles)
            if d.ndim == 2:
                d = d[None]
            d = np.ascontiguousarray(d)
        C = q.shape[0] if q is not None else d.shape[0]
        ns = self._npoints(0)
        nt = self._npoints(1)
        if q is not None and q.shape != (C, ns):
            raise ValueError("charges must be (C, Ns) or (Ns,)")
        if d is not None and d.shape != (C, ns, 3):
            raise ValueError("dipoles must be (C, Ns, 3) or (Ns, 3)")
        pot = np.zeros((C, nt))
        grad = np.zeros((C, nt, 3)) if want_gradient else None
        if C in (1, 4, 7):
            self._eval_block(q, d, C, p, want_gradient, parts, pot, grad)
        else:  # run in single channels
            for c in range(C):
                gp = np.zeros((1, nt))
                gg = np.zeros((1, nt, 3)) if want_gradient else None
                self._eval_block(None if q is None else q[c:c + 1], None if d is None else d[c:c + 1],
                                 1, p, want_gradient, parts, gp, gg)
                pot[c] = gp[0]
                if want_gradient:
                    grad[c] = gg[0]
        if single:
            return (pot[0], grad[0]) if want_gradient else pot[0]
        return (pot, grad) if want_gradient else pot

    def _eval_block(self, q, d, C, p, want_gradient, parts, pot, grad):
        qq = None if q is None else np.ascontiguousarray(q)
        dd = None if d is None else np.ascontiguousarray(d)
        N.check(self._lib.fmmbem_plan_evaluate(
            self._h, None if qq is None else N.dptr(qq), None if dd is None else N.dptr(dd), C,
            int(p), 1 if want_gradient else 0, parts, N.dptr(pot),
            N.dptr(grad) if grad is not None else None))

    def far_field(self, charges=None, dipoles=None, p=8, want_gradient=False):
        """``FmmPlan.far_field`` (fmm.py:203-233): expansion part only, no 1/(4 pi)."""
        return self._evaluate(charges, dipoles, p, want_gradient, 1)

    def near_field(self, charges=None, dipoles=None, want_gradient=False):
        """``FmmPlan.near_field`` (fmm.py:356-419): direct sums over the P2P pairs."""
        return self._evaluate(charges, dipoles, 0, want_gradient, 2)


class GpuBemOperator:
    """``BemOperator`` (bemop.py:43-315) with every layer application on the device."""

    def __init__(self, mesh, formulation, theta=0.5, n_crit=126, mu=1e-3, near_factor=2.0,
                 n_gauss_singular=32, device=0, max_depth=20):
        self._lib = N.load()
        self.mesh = mesh
        self.formulation = _formulation(formulation)
        self.mu = mu
        self.theta = theta
        self.n_crit = n_crit
        self.near_factor = near_factor
        self.device = device
        if not 0.0 < theta < 1.0:
            raise ValueError("theta must be in (0, 1)")
        if n_crit < 1:
            raise ValueError("n_crit must be >= 1")
        ps = PanelSet(mesh)
        self._panels = ps
        self.normals = ps.normals
        self.areas = ps.areas
        self.centroids = ps.centroids
        self.src_pos = ps.src_pos
        self.src_weight = ps.src_weight
        self.src_panel = np.repeat(np.arange(ps.n_panels), 4)
        self.src_normal = np.repeat(self.normals, 4, axis=0)
        lx, lw = gauss_legendre(int(n_gauss_singular))
        gp = np.ascontiguousarray(ps.src_pos.reshape(ps.n_panels, 4, 3))
        gw = np.ascontiguousarray(ps.src_weight.reshape(ps.n_panels, 4))
        h = ctypes.c_void_p()
        N.check(self._lib.fmmbem_op_create(
            N.dptr(ps.panel_vertices), ps.n_panels, N.dptr(gp), N.dptr(gw), N.dptr(ps.fine_pos),
            N.dptr(ps.fine_weight), N.dptr(ps.normals), N.dptr(ps.areas), N.dptr(lx), N.dptr(lw),
            int(n_gauss_singular), _FORM_CODE[self.formulation], float(theta), int(n_crit),
            float(mu), float(near_factor), int(max_depth), int(device), ctypes.byref(h)))
        self._h = h
        n = ctypes.c_int64(0)
        N.check(self._lib.fmmbem_op_size(self._h, ctypes.byref(n)))
        self._n = int(n.value)
        ph = ctypes.c_void_p()
        N.check(self._lib.fmmbem_op_plan(self._h, ctypes.byref(ph)))
        self.plan = GpuFmmPlan(None, None, n_crit=n_crit, theta=theta, device=device, _handle=ph,
                               _owner=self)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.fmmbem_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_panels(self) -> int:
        return self._panels.n_panels

    @property
    def shape(self):
        return (self._n, self._n)

    def _vec(self, x):
        v = N.f64(np.asarray(x, dtype=float).reshape(-1))
        if v.shape != (self._n,):
            raise ValueError(f"expected a vector of length {self._n}, got {v.shape}")
        return v

    def apply(self, x, p=12):
        """System mat-vec A x with expansions truncated at order p (bemop.py:272-274)."""
        v = self._vec(x)
        y = N.host_array(self._n)
        N.check(self._lib.fmmbem_op_apply(self._h, N.dptr(v), N.dptr(y), int(p)))
        return y

    def apply_device(self, x_ptr: int, y_ptr: int, p: int = 12, stream: int | None = None):
        """Device-pointer mat-vec (raw CUDA addresses of n float64 each).

        ``stream`` (a raw cudaStream_t, e.g. ``torch.cuda.current_stream().cuda_stream``):
        the apply is ordered after the work queued there and the stream waits for it; the call
        returns without a host synchronisation.  ``None``: ordered after the legacy default
        stream, synchronous."""
        N.check(self._lib.fmmbem_op_apply_device(self._h, ctypes.c_void_p(x_ptr),
                                                 ctypes.c_void_p(y_ptr), int(p),
                                                 None if stream is None else ctypes.c_void_p(stream)))

    def dense_apply(self, x):
        """Direct-sum mat-vec (bemop.py:276-278)."""
        v = self._vec(x)
        y = np.empty(self._n)
        N.check(self._lib.fmmbem_op_dense_apply(self._h, N.dptr(v), N.dptr(y)))
        return y

    def assemble_rhs(self, boundary_data, p=18, dense=None):
        """Right-hand side from the boundary data (bemop.py:290-310)."""
        if dense is None:
            dense = self._n <= 8192
        v = self._vec(boundary_data)
        b = np.empty(self._n)
        N.check(self._lib.fmmbem_op_assemble_rhs(self._h, N.dptr(v), int(p), 1 if dense else 0,
                                                 N.dptr(b)))
        return b

    def drag_force(self, traction):
        """Net force sum_j area_j t_j (bemop.py:312-315)."""
        t = np.asarray(traction, dtype=float).reshape(self.n_panels, 3)
        return np.einsum("p,pi->i", self.areas, t)

    def correction(self, which: str = "sys"):
        """(indptr, indices, data, block) of C_sys / C_rhs as assembled on the device."""
        w = 0 if which == "sys" else 1
        nnz = ctypes.c_int64(0)
        blk = ctypes.c_int32(0)
        N.check(self._lib.fmmbem_op_correction(self._h, w, ctypes.byref(nnz), ctypes.byref(blk),
                                               None, None, None))
        indptr = np.empty(self.n_panels + 1, np.int64)
        indices = np.empty(nnz.value, np.int64)
        data = np.empty(nnz.value * blk.value)
        N.check(self._lib.fmmbem_op_correction(self._h, w, None, None, N.i64ptr(indptr),
                                               N.i64ptr(indices), N.dptr(data)))
        return indptr, indices, data, int(blk.value)

    def set_timing(self, enable: bool, use_graphs: bool = True):
        N.check(self._lib.fmmbem_op_set_timing(self._h, 1 if enable else 0, 1 if use_graphs else 0))

    def set_serial(self, serial: bool):
        """Run the near field in line with the far field (isolated kernel timings)."""
        N.check(self._lib.fmmbem_op_set_serial(self._h, 1 if serial else 0))

    # -- multi-GPU ---------------------------------------------------------------
    def leaf_work(self, which: str = "tgt") -> np.ndarray:
        """Per-leaf work weights (body order) used to partition the leaves across ranks."""
        w = np.zeros(self.plan.n_tgt_leaves if which == "tgt" else self.plan.n_src_leaves)
        N.check(self._lib.fmmbem_op_leaf_work(self._h, 0 if which == "tgt" else 1, N.dptr(w)))
        return w

    def shard(self, rank: int, world: int, tleaf_bounds, sleaf_bounds, nccl_id: bytes | None = None):
        """Own target leaves [tb[rank], tb[rank+1]) and source leaves [sb[rank], sb[rank+1]).

        nccl_id: 128 bytes shared by all ranks (``nccl_unique_id()`` on rank 0); None makes a
        "virtual" shard that computes only its own rows without collectives (testing).
        """
        tb = np.ascontiguousarray(tleaf_bounds, dtype=np.int32)
        sb = np.ascontiguousarray(sleaf_bounds, dtype=np.int32)
        if tb.shape != (world + 1,) or sb.shape != (world + 1,):
            raise ValueError("bounds must have world + 1 entries")
        if nccl_id is not None and len(nccl_id) != 128:
            raise ValueError("nccl_id must be 128 bytes")
        N.check(self._lib.fmmbem_op_shard(self._h, int(rank), int(world), N.i32ptr(tb), N.i32ptr(sb),
                                          nccl_id))

    def shard_host(self, rank: int, world: int, tleaf_bounds, sleaf_bounds, allgather, allreduce):
        """The same partition over a HOST transport: ``allgather(send) -> recv`` (numpy
        float64, recv = every rank's send concatenated in rank order) and ``allreduce(buf)``
        (in-place sum) are called for every collective of the sharded apply / GMRES."""
        tb = np.ascontiguousarray(tleaf_bounds, dtype=np.int32)
        sb = np.ascontiguousarray(sleaf_bounds, dtype=np.int32)
        if tb.shape != (world + 1,) or sb.shape != (world + 1,):
            raise ValueError("bounds must have world + 1 entries")

        def _ag(send_p, recv_p, count, _user):
            try:
                send = np.ctypeslib.as_array(send_p, shape=(count,))
                recv = np.ctypeslib.as_array(recv_p, shape=(world * count,))
                recv[:] = np.asarray(allgather(send.copy()), dtype=np.float64).reshape(-1)
                return 0
            except BaseException:  # reported as a CUDA-side failure of the collective
                return 1

        def _ar(buf_p, count, _user):
            try:
                buf = np.ctypeslib.as_array(buf_p, shape=(count,))
                buf[:] = np.asarray(allreduce(buf.copy()), dtype=np.float64).reshape(-1)
                return 0
            except BaseException:
                return 1

        # the ctypes thunks must outlive the shard
        self._host_cbs = (N.ALLGATHER_CALLBACK(_ag), N.ALLREDUCE_CALLBACK(_ar))
        N.check(self._lib.fmmbem_op_shard_host(self._h, int(rank), int(world), N.i32ptr(tb),
                                               N.i32ptr(sb), self._host_cbs[0],
                                               self._host_cbs[1], None))

    def unshard(self):
        N.check(self._lib.fmmbem_op_unshard(self._h))
        self._host_cbs = None

    def owned_panels(self, tleaf_bounds, rank: int) -> np.ndarray:
        """Panel indices whose rows rank `rank` computes under the given target split."""
        t = self.plan.tree("tgt")
        leaves = np.flatnonzero(t["is_leaf"])
        leaves = leaves[np.argsort(t["body_start"][leaves], kind="stable")]
        a, b = int(tleaf_bounds[rank]), int(tleaf_bounds[rank + 1])
        if a == b:
            return np.zeros(0, dtype=np.int64)
        s0 = t["body_start"][leaves[a]]
        s1 = t["body_start"][leaves[b - 1]] + t["body_count"][leaves[b - 1]]
        return np.sort(t["perm"][s0:s1])

    def counters(self):
        """(kernel launches so far, graph applies so far, last GMRES call device ms)."""
        kl = ctypes.c_int64(0)
        ap = ctypes.c_int64(0)
        ms = ctypes.c_double(0.0)
        N.check(self._lib.fmmbem_op_counters(self._h, ctypes.byref(kl), ctypes.byref(ap),
                                             ctypes.byref(ms)))
        return int(kl.value), int(ap.value), float(ms.value)

    def stage_times(self, reset: bool = False):
        """Accumulated CUDA-event ms per stage: p2p, p2m+m2m, m2l, l2l, epilogue, total."""
        ms = np.zeros(6)
        calls = ctypes.c_int64(0)
        N.check(self._lib.fmmbem_op_stage_times(self._h, N.dptr(ms), ctypes.byref(calls),
                                                1 if reset else 0))
        keys = ("p2p", "p2m_m2m", "m2l", "l2l", "epilogue", "total")
        return dict(zip(keys, ms.tolist())), int(calls.value)
