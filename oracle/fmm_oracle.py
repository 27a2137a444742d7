"""numpy/scipy restatement of the reference FMM-BEM hot path (TEST INFRASTRUCTURE).

Every function names the reference code it restates (paths relative to
/root/reference/pkg/src/fmmbem).  Pinned against goldens produced by the
reference itself (tests/golden, tests/test_oracle.py).  Used by the tests,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs only.

Coefficients use the reference's full flat layout n*n + n + m (harmonics.py:
30-35), deliberately unlike the device code's half storage, so the two
implementations share no indexing code.
"""

from __future__ import annotations

import math
import os
import sys
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
from scipy.spatial import cKDTree

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_1506_05957_b200.geometry import PanelSet, gauss_legendre  # noqa: E402  (input prep)

FOUR_PI = 4.0 * np.pi
EIGHT_PI = 8.0 * np.pi


def nco(p):
    return (p + 1) * (p + 1)


def fidx(n, m):
    return n * n + n + m


# --------------------------------------------------------------- harmonics
def solid_harmonics(v, p, irregular=False):
    """R_n^m (regular, harmonics.py:38-59) or I_n^m (irregular, :62-85), full layout.

    Built column by column in m from the sectoral term with a two-term
    recurrence in n; negative orders by (-1)^m conj.
    """
    v = np.atleast_2d(np.asarray(v, dtype=float))
    x, y, z = v[:, 0], v[:, 1], v[:, 2]
    r2 = x * x + y * y + z * z
    w = x + 1j * y
    out = np.zeros((len(v), nco(p)), dtype=complex)
    sect = np.ones(len(v), dtype=complex) if not irregular else (1.0 / np.sqrt(r2)).astype(complex)
    for m in range(p + 1):
        if m:
            sect = sect * (-(2 * m - 1) * w / r2 if irregular else -w / (2 * m))
        col_prev, col = None, sect
        for n in range(m, p + 1):
            if n == m + 1:
                col_prev, col = col, (((2 * m + 1) * z / r2) if irregular else z) * col
            elif n > m + 1:
                if irregular:
                    nxt = ((2 * n - 1) * z * col - ((n - 1) ** 2 - m * m) * col_prev) / r2
                else:
                    nxt = ((2 * n - 1) * z * col - r2 * col_prev) / ((n + m) * (n - m))
                col_prev, col = col, nxt
            out[:, fidx(n, m)] = col
            if m:
                out[:, fidx(n, -m)] = (-1) ** m * np.conj(col)
    return out


def _shift(arr, p, dn, dm):
    """Entry (n, m) <- arr[(n + dn, m + dm)] within order p (0 where undefined)."""
    out = np.zeros_like(arr)
    for n in range(p + 1):
        for m in range(-n, n + 1):
            nn, mm = n + dn, m + dm
            if 0 <= nn <= p and abs(mm) <= nn:
                out[..., fidx(n, m)] = arr[..., fidx(nn, mm)]
    return out


def regular_grad(R, p):
    """(d/dx, d/dy, d/dz) of R_n^m via the shift rules (harmonics.py:128-140)."""
    a = _shift(R, p, -1, +1)     # (dx + i dy) R_n^m = R_{n-1}^{m+1}
    b = -_shift(R, p, -1, -1)    # (dx - i dy) R_n^m = -R_{n-1}^{m-1}
    return 0.5 * (a + b), (a - b) / 2j, _shift(R, p, -1, 0)


def _mat_rconv(Rd, p, kind):
    """Dense M2M / L2L operator from R(d) (harmonics.py:156-177, 201-218)."""
    T = np.zeros((nco(p), nco(p)), dtype=complex)
    for n in range(p + 1):
        for m in range(-n, n + 1):
            o = fidx(n, m)
            for j in range(p + 1):
                for k in range(-j, j + 1):
                    if kind == "m2m" and j <= n and abs(m - k) <= n - j:
                        T[o, fidx(j, k)] = Rd[fidx(n - j, m - k)]
                    if kind == "l2l" and j >= n and abs(k - m) <= j - n:
                        T[o, fidx(j, k)] = Rd[fidx(j - n, k - m)]
    return T


_M2L_CACHE = {}


def _m2l_gather(p):
    """(index map into I of order 2p, sign) for M2L (harmonics.py:180-198)."""
    if p not in _M2L_CACHE:
        g = np.empty((nco(p), nco(p)), dtype=np.intp)
        s = np.empty(nco(p))
        for j in range(p + 1):
            for k in range(-j, j + 1):
                s[fidx(j, k)] = -1.0 if j % 2 else 1.0
                for n in range(p + 1):
                    for m in range(-n, n + 1):
                        g[fidx(j, k), fidx(n, m)] = fidx(n + j, m + k)
        _M2L_CACHE[p] = (g, s)
    return _M2L_CACHE[p]


# --------------------------------------------------------------- octree
@dataclass
class Tree:
    points: np.ndarray
    perm: np.ndarray
    center: np.ndarray
    half: np.ndarray
    level: np.ndarray
    parent: np.ndarray
    children: list
    start: np.ndarray
    count: np.ndarray

    @property
    def is_leaf(self):
        return np.array([len(c) == 0 for c in self.children])

    @property
    def leaves(self):
        lv = np.flatnonzero(self.is_leaf)
        return lv[np.argsort(self.start[lv], kind="stable")]


def bounding_cube(points, pad=1e-6):
    """octree.py:46-54."""
    lo, hi = points.min(axis=0), points.max(axis=0)
    half = 0.5 * float(np.max(hi - lo))
    return 0.5 * (lo + hi), half * (1.0 + pad) + pad


def build_tree(points, n_crit, center, half, max_depth=20):
    """Adaptive octree of octree.py:57-131 (split when count > n_crit and level < max_depth,
    octant by strict '>' against the cell centre, child centre c +- h, DFS numbering with
    octant 0 first, input order kept inside leaves).  Restated with an explicit work list
    over index arrays."""
    pts = np.asarray(points, dtype=float)
    cells = []   # dicts
    order = []   # output body order
    work = [(np.asarray(center, float), float(half), 0, -1, np.arange(len(pts)))]
    while work:
        c, h, lev, par, idx = work.pop()
        cid = len(cells)
        cells.append(dict(center=c, half=h, level=lev, parent=par, kids=[], idx=idx))
        if par >= 0:
            cells[par]["kids"].append(cid)
        if len(idx) <= n_crit or lev >= max_depth:
            cells[cid]["start"] = len(order)
            order.extend(idx.tolist())
            continue
        oc = ((pts[idx, 0] > c[0]).astype(int) + 2 * (pts[idx, 1] > c[1]) + 4 * (pts[idx, 2] > c[2]))
        hh = h * 0.5
        sub = []
        for o in range(8):
            sel = idx[oc == o]
            if len(sel):
                off = np.array([hh if o & 1 else -hh, hh if o & 2 else -hh, hh if o & 4 else -hh])
                sub.append((c + off, hh, lev + 1, cid, sel))
        work.extend(reversed(sub))
    n = len(cells)
    start = np.zeros(n, dtype=np.intp)
    for k in range(n - 1, -1, -1):
        start[k] = cells[k]["start"] if not cells[k]["kids"] else min(start[j] for j in cells[k]["kids"])
    return Tree(points=pts, perm=np.asarray(order, dtype=np.intp),
                center=np.array([c["center"] for c in cells]), half=np.array([c["half"] for c in cells]),
                level=np.array([c["level"] for c in cells]), parent=np.array([c["parent"] for c in cells]),
                children=[c["kids"] for c in cells], start=start,
                count=np.array([len(c["idx"]) for c in cells]))


def dual_traversal(S: Tree, T: Tree, theta):
    """fmm.py:84-125 with CELL_RADIUS_FACTOR = 1 (r = half width)."""
    m2l, p2p = [], []
    s_leaf, t_leaf = S.is_leaf, T.is_leaf
    stack = [(0, 0)]
    while stack:
        s, t = stack.pop()
        d = math.dist(S.center[s], T.center[t])
        if d > 0.0 and (S.half[s] + T.half[t]) < theta * d:
            m2l.append((s, t))
            continue
        if s_leaf[s] and t_leaf[t]:
            p2p.append((s, t))
            continue
        if not s_leaf[s] and (t_leaf[t] or S.half[s] >= T.half[t]):
            stack.extend((k, t) for k in S.children[s])
        else:
            stack.extend((s, k) for k in T.children[t])
    return np.array(m2l, dtype=np.intp).reshape(-1, 2), np.array(p2p, dtype=np.intp).reshape(-1, 2)


# --------------------------------------------------------------- FMM
class OraclePlan:
    """FmmPlan (fmm.py:128-419), policy 'fmm'."""

    def __init__(self, src, tgt, n_crit=126, theta=0.5, max_depth=20):
        src = np.atleast_2d(np.asarray(src, float))
        tgt = np.atleast_2d(np.asarray(tgt, float))
        c, h = bounding_cube(np.vstack([src, tgt]))
        self.S = build_tree(src, n_crit, c, h, max_depth)
        self.T = build_tree(tgt, n_crit, c, h, max_depth)
        self.m2l_pairs, self.p2p_pairs = dual_traversal(self.S, self.T, theta)
        self.root_half = h
        self._igrid = {}
        self._vert = {}
        # near lists per target leaf (fmm.py:161-167)
        self.near = {}
        for s, t in self.p2p_pairs:
            self.near.setdefault(int(t), []).append(int(s))

    def _bodies(self, tree, c):
        return tree.perm[tree.start[c]:tree.start[c] + tree.count[c]]

    def _operators(self, tree, p, kind):
        key = (id(tree), p, kind)
        if key not in self._vert:
            ops = {}
            for c in range(1, len(tree.center)):
                d = tree.center[c] - tree.center[tree.parent[c]]
                k = (int(tree.level[c]), tuple(np.sign(d).astype(int)))
                if k not in ops:
                    ops[k] = _mat_rconv(solid_harmonics(d[None], p)[0], p, kind)
            self._vert[key] = ops
        return self._vert[key]

    def far_field(self, charges=None, dipoles=None, p=8, want_gradient=False):
        """P2M -> M2M -> M2L -> L2L -> L2P (fmm.py:203-336); no P2P, no 1/(4 pi)."""
        S, T = self.S, self.T
        q = None if charges is None else np.atleast_2d(np.asarray(charges, float))
        d = None if dipoles is None else np.asarray(dipoles, float)
        if d is not None and d.ndim == 2:
            d = d[None]
        C = q.shape[0] if q is not None else d.shape[0]
        M = np.zeros((len(S.center), C, nco(p)), dtype=complex)
        for leaf in S.leaves:
            b = self._bodies(S, leaf)
            R = solid_harmonics(S.points[b] - S.center[leaf], p)
            if q is not None:
                M[leaf] += q[:, b] @ R
            if d is not None:
                gx, gy, gz = regular_grad(R, p)
                M[leaf] += d[:, b, 0] @ gx + d[:, b, 1] @ gy + d[:, b, 2] @ gz
        up = self._operators(S, p, "m2m")
        for lev in range(int(S.level.max()), 0, -1):
            for c in np.flatnonzero(S.level == lev):
                dd = S.center[c] - S.center[S.parent[c]]
                Tm = up[(lev, tuple(np.sign(dd).astype(int)))]
                M[S.parent[c]] += M[c] @ Tm.T
        L = np.zeros((len(T.center), C, nco(p)), dtype=complex)
        if len(self.m2l_pairs):
            g, sg = _m2l_gather(p)
            Dq = T.center[self.m2l_pairs[:, 1]] - S.center[self.m2l_pairs[:, 0]]
            # offsets are lattice vectors; the reference rounds to half * 2^-22 (fmm.py:144-151)
            quantum = self.root_half * 2.0 ** -22
            keys = np.round(Dq / quantum).astype(np.int64)
            uk, inv = np.unique(keys, axis=0, return_inverse=True)
            inv = inv.ravel()
            if p not in self._igrid:
                self._igrid[p] = solid_harmonics(uk * quantum, 2 * p, irregular=True)
            Ig = self._igrid[p]
            for u in range(len(uk)):
                sel = np.flatnonzero(inv == u)
                Tm = sg[:, None] * np.conj(Ig[u][g])
                src, tgt = self.m2l_pairs[sel, 0], self.m2l_pairs[sel, 1]
                L[tgt] += (M[src].reshape(-1, nco(p)) @ Tm.T).reshape(len(sel), C, nco(p))
        down = self._operators(T, p, "l2l")
        for lev in range(1, int(T.level.max()) + 1):
            for c in np.flatnonzero(T.level == lev):
                dd = T.center[c] - T.center[T.parent[c]]
                Tm = down[(lev, tuple(np.sign(dd).astype(int)))]
                L[c] += L[T.parent[c]] @ Tm.T
        nt = len(T.points)
        pot = np.zeros((C, nt))
        grad = np.zeros((C, nt, 3)) if want_gradient else None
        for leaf in T.leaves:
            b = self._bodies(T, leaf)
            R = solid_harmonics(T.points[b] - T.center[leaf], p)
            pot[:, b] += np.real(L[leaf] @ R.T)
            if want_gradient:
                for k, gk in enumerate(regular_grad(R, p)):
                    grad[:, b, k] += np.real(L[leaf] @ gk.T)
        single = (charges is not None and np.asarray(charges).ndim == 1) or (
            charges is None and np.asarray(dipoles).ndim == 2)
        if single:
            return (pot[0], grad[0]) if want_gradient else pot[0]
        return (pot, grad) if want_gradient else pot

    def near_field(self, charges=None, dipoles=None, want_gradient=False):
        """Direct sums over the P2P lists, coincident pairs zero (fmm.py:356-419)."""
        S, T = self.S, self.T
        q = None if charges is None else np.atleast_2d(np.asarray(charges, float))
        d = None if dipoles is None else np.asarray(dipoles, float)
        if d is not None and d.ndim == 2:
            d = d[None]
        C = q.shape[0] if q is not None else d.shape[0]
        nt = len(T.points)
        pot = np.zeros((C, nt))
        grad = np.zeros((C, nt, 3)) if want_gradient else None
        for t, srcs in self.near.items():
            ti = self._bodies(T, t)
            si = np.sort(np.concatenate([self._bodies(S, s) for s in srcs]))
            r = T.points[ti][:, None, :] - S.points[si][None, :, :]
            r2 = np.einsum("abk,abk->ab", r, r)
            inv = np.where(r2 > 0.0, 1.0 / np.sqrt(np.where(r2 > 0.0, r2, 1.0)), 0.0)
            i3 = inv ** 3
            if q is not None:
                pot[:, ti] += q[:, si] @ inv.T
                if want_gradient:
                    grad[:, ti] -= np.einsum("cs,tsk,ts->ctk", q[:, si], r, i3)
            if d is not None:
                rd = np.einsum("tsk,csk->cts", r, d[:, si])
                pot[:, ti] += np.einsum("cts,ts->ct", rd, i3)
                if want_gradient:
                    grad[:, ti] += np.einsum("csk,ts->ctk", d[:, si], i3)
                    grad[:, ti] -= 3.0 * np.einsum("cts,tsk,ts->ctk", rd, r, i3 * inv * inv)
        single = (charges is not None and np.asarray(charges).ndim == 1) or (
            charges is None and np.asarray(dipoles).ndim == 2)
        if single:
            return (pot[0], grad[0]) if want_gradient else pot[0]
        return (pot, grad) if want_gradient else pot


# --------------------------------------------------------------- BEM operator
KERNELS = ("laplace_single", "laplace_double", "stokeslet", "stresslet")


def rule_sum(kind, x, pts, wts, nrm):
    """Per-pair rule sums (bemop.py:104-125): x (Np,3), pts (Np,K,3), wts (Np,K), nrm (Np,3)."""
    r = x[:, None, :] - pts
    r2 = np.einsum("pki,pki->pk", r, r)
    inv = np.where(r2 > 0.0, 1.0 / np.sqrt(np.where(r2 > 0.0, r2, 1.0)), 0.0)
    if kind == "laplace_single":
        return (wts * inv).sum(axis=1) / FOUR_PI
    if kind == "laplace_double":
        return (wts * np.einsum("pki,pi->pk", r, nrm) * inv ** 3).sum(axis=1) / FOUR_PI
    if kind == "stokeslet":
        blk = np.einsum("pk,pki,pkj->pij", wts * inv ** 3, r, r)
        return blk + np.eye(3)[None] * (wts * inv).sum(axis=1)[:, None, None]
    rn = np.einsum("pki,pi->pk", r, nrm)
    return 6.0 * np.einsum("pk,pki,pkj->pij", wts * rn * inv ** 5, r, r)


def singular_self(kind, v, n_gauss):
    """Hess-Smith polar integral about the centroid (quadrature.py:175-247)."""
    cen = v.mean(axis=0)
    nrm = np.cross(v[1] - v[0], v[2] - v[0])
    nrm = nrm / np.linalg.norm(nrm)
    e1 = (v[1] - v[0]) - np.dot(v[1] - v[0], nrm) * nrm
    e1 = e1 / np.linalg.norm(e1)
    e2 = np.cross(nrm, e1)
    uv = np.stack([(v - cen) @ e1, (v - cen) @ e2], axis=1)
    gx, gw = gauss_legendre(n_gauss)
    tot, b = 0.0, np.zeros((2, 2))
    for i in range(3):
        a, c = uv[i], uv[(i + 1) % 3]
        t0, t1 = math.atan2(a[1], a[0]), math.atan2(c[1], c[0])
        if t1 <= t0:
            t1 += 2.0 * math.pi
        phi = 0.5 * (t1 - t0) * gx + 0.5 * (t1 + t0)
        wp = 0.5 * (t1 - t0) * gw
        ne = np.array([c[1] - a[1], a[0] - c[0]])
        ne = ne / np.linalg.norm(ne)
        de = float(ne @ a)
        if de < 0.0:
            ne, de = -ne, -de
        R = de / (np.cos(phi) * ne[0] + np.sin(phi) * ne[1])
        tot += float(wp @ R)
        cs, sn = np.cos(phi), np.sin(phi)
        b += np.array([[wp @ (R * cs * cs), wp @ (R * cs * sn)], [wp @ (R * cs * sn), wp @ (R * sn * sn)]])
    if kind == "laplace_single":
        return tot / FOUR_PI
    loc = np.eye(3) * tot
    loc[:2, :2] += b
    F = np.stack([e1, e2, nrm])
    return F.T @ loc @ F


class OracleOperator:
    """BemOperator (bemop.py:43-315): apply / dense_apply / assemble_rhs / drag."""

    def __init__(self, mesh, formulation, theta=0.5, n_crit=126, mu=1e-3, near_factor=2.0,
                 n_gauss_singular=32, plan=True):
        self.formulation = getattr(formulation, "value", formulation)
        self.mu = mu
        ps = PanelSet(mesh)
        self.ps = ps
        self.P = ps.n_panels
        self.n = 3 * self.P if self.formulation == "stokes" else self.P
        self.centroids, self.normals, self.areas = ps.centroids, ps.normals, ps.areas
        self.src_pos, self.src_weight = ps.src_pos, ps.src_weight
        self.src_panel = np.repeat(np.arange(self.P), 4)
        self.src_normal = np.repeat(self.normals, 4, axis=0)
        self.plan = OraclePlan(self.src_pos, self.centroids, n_crit, theta) if plan else None
        cut = near_factor * np.sqrt(2.0 * self.areas)
        hits = cKDTree(self.centroids).query_ball_point(self.centroids, cut, return_sorted=True)
        self.near_pairs = np.array([(i, j) for j, h in enumerate(hits) for i in h],
                                   dtype=np.intp).reshape(-1, 2)
        stokes = self.formulation == "stokes"
        sysk, rhsk = ("stokeslet", "stresslet") if stokes else ("laplace_single", "laplace_double")
        if self.formulation == "laplace_second":
            sysk, rhsk = rhsk, sysk
        self.sys_kind, self.rhs_kind = sysk, rhsk
        self.c_sys = self._correction(sysk, n_gauss_singular)
        self.c_rhs = self._correction(rhsk, n_gauss_singular)

    def _correction(self, kind, ng):
        """bemop.py:127-184."""
        ps = self.ps
        ti, sj = self.near_pairs[:, 0], self.near_pairs[:, 1]
        x = self.centroids[ti]
        nj = self.normals[sj]
        coarse = rule_sum(kind, x, ps.src_pos.reshape(-1, 4, 3)[sj], ps.src_weight.reshape(-1, 4)[sj], nj)
        fine = rule_sum(kind, x, ps.fine_pos[sj], ps.fine_weight[sj], nj)
        delta = fine - coarse
        for s in np.flatnonzero(ti == sj):
            j = sj[s]
            if kind in ("laplace_single", "stokeslet"):
                delta[s] = delta[s] + singular_self(kind, ps.panel_vertices[j], ng)
            delta[s] = delta[s] - fine[s]
        n = self.n
        if kind in ("laplace_single", "laplace_double"):
            return sp.csr_matrix((delta, (ti, sj)), shape=(n, n))
        a, b = np.meshgrid(np.arange(3), np.arange(3), indexing="ij")
        rows = (3 * ti[:, None, None] + a[None]).ravel()
        cols = (3 * sj[:, None, None] + b[None]).ravel()
        return sp.csr_matrix((delta.ravel(), (rows, cols)), shape=(n, n))

    def _dense(self, q, d, want_gradient):
        """All-pairs sums (bemop.py:234-268)."""
        C = q.shape[0] if q is not None else d.shape[0]
        nt = self.P
        pot = np.zeros((C, nt))
        grad = np.zeros((C, nt, 3)) if want_gradient else None
        for lo in range(0, nt, 256):
            tg = self.centroids[lo:lo + 256]
            r = tg[:, None, :] - self.src_pos[None]
            r2 = np.einsum("tsk,tsk->ts", r, r)
            inv = np.where(r2 > 0.0, 1.0 / np.sqrt(np.where(r2 > 0.0, r2, 1.0)), 0.0)
            i3 = inv ** 3
            sl = slice(lo, lo + len(tg))
            if q is not None:
                pot[:, sl] += q @ inv.T
                if want_gradient:
                    grad[:, sl] -= np.einsum("cs,tsk,ts->ctk", q, r, i3)
            if d is not None:
                rd = np.einsum("tsk,csk->cts", r, d)
                pot[:, sl] += np.einsum("cts,ts->ct", rd, i3)
                if want_gradient:
                    grad[:, sl] += np.einsum("csk,ts->ctk", d, i3)
                    grad[:, sl] -= 3.0 * np.einsum("cts,tsk,ts->ctk", rd, r, i3 * inv * inv)
        return pot, grad

    def layer(self, kind, x, p, corr, dense=False):
        """bemop.py:192-232."""
        x = np.asarray(x, float)
        if kind in ("laplace_single", "laplace_double"):
            s = self.src_weight * x[self.src_panel]
            q, d = (s[None], None) if kind == "laplace_single" else (None, (s[:, None] * self.src_normal)[None])
            if dense:
                out = self._dense(q, d, False)[0][0]
            else:
                out = self.plan.far_field(charges=q, dipoles=d, p=p)[0] + \
                    self.plan.near_field(charges=q, dipoles=d)[0]
            return out / FOUR_PI + corr @ x
        f = self.src_weight[:, None] * x.reshape(self.P, 3)[self.src_panel]
        y = self.src_pos
        X = self.centroids
        if kind == "stokeslet":
            q = np.vstack([f.T, np.einsum("si,si->s", y, f)])    # fmm.py:422-425
            if dense:
                pot, grad = self._dense(q, None, True)
            else:
                pot, grad = self.plan.far_field(charges=q, p=p, want_gradient=True)
                npot, ngrad = self.plan.near_field(charges=q, want_gradient=True)
                pot, grad = pot + npot, grad + ngrad
            u = pot[:3].T - np.einsum("tc,cti->ti", X, grad[:3]) + grad[3]   # fmm.py:428-433
        else:
            nn = self.src_normal
            d = np.empty((7, len(f), 3))                          # fmm.py:436-445
            for c in range(3):
                d[c] = f[:, c:c + 1] * nn
                d[3 + c] = nn[:, c:c + 1] * f
            d[6] = np.einsum("si,si->s", y, f)[:, None] * nn
            if dense:
                pot, grad = self._dense(None, d, True)
            else:
                pot, grad = self.plan.far_field(dipoles=d, p=p, want_gradient=True)
                npot, ngrad = self.plan.near_field(dipoles=d, want_gradient=True)
                pot, grad = pot + npot, grad + ngrad
            u = 2.0 * pot[3:6].T - 2.0 * np.einsum("tc,cti->ti", X, grad[:3]) + 2.0 * grad[6]
        return u.reshape(-1) + corr @ x

    def _apply(self, x, p, dense):
        """bemop.py:280-288."""
        if self.formulation == "laplace_first":
            return self.layer("laplace_single", x, p, self.c_sys, dense)
        if self.formulation == "laplace_second":
            return 0.5 * np.asarray(x, float) - self.layer("laplace_double", x, p, self.c_sys, dense)
        return self.layer("stokeslet", x, p, self.c_sys, dense) / (EIGHT_PI * self.mu)

    def apply(self, x, p=12):
        return self._apply(x, p, False)

    def dense_apply(self, x):
        return self._apply(x, 0, True)

    def assemble_rhs(self, data, p=18, dense=None):
        """bemop.py:290-310."""
        if dense is None:
            dense = self.n <= 8192
        data = np.asarray(data, float).reshape(-1)
        if self.formulation == "laplace_first":
            return 0.5 * data - self.layer("laplace_double", data, p, self.c_rhs, dense)
        if self.formulation == "laplace_second":
            return self.layer("laplace_single", data, p, self.c_rhs, dense)
        return 0.5 * data - self.layer("stresslet", data, p, self.c_rhs, dense) / EIGHT_PI


# --------------------------------------------------------------- GMRES
@dataclass
class RelaxationSchedule:
    """solver.py:20-47."""
    p_initial: int = 12
    p_min: int = 1
    eta: float = 1e-5
    relaxed: bool = True

    def order(self, r, prev):
        if not self.relaxed:
            return self.p_initial
        eps = min(self.eta / min(max(r, self.eta), 1.0), 1.0)
        p = math.ceil(-math.log2(eps)) if eps < 1.0 else self.p_min
        return min(int(min(self.p_initial, max(self.p_min, p))), prev)


@dataclass
class Result:
    x: np.ndarray
    residuals: list = field(default_factory=list)
    orders: list = field(default_factory=list)
    converged: bool = False

    @property
    def n_iterations(self):
        return len(self.orders)


def gmres(apply_fn, b, schedule, tol, max_iter):
    """Unrestarted MGS-Arnoldi GMRES with Givens rotations (solver.py:69-134)."""
    b = np.asarray(b, float)
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return Result(np.zeros_like(b), converged=True)
    V = [b / nb]
    H = np.zeros((max_iter + 1, max_iter))
    cs, sn = np.zeros(max_iter), np.zeros(max_iter)
    g = np.zeros(max_iter + 1)
    g[0] = nb
    out = Result(np.zeros_like(b))
    r, prev = 1.0, schedule.p_initial
    for k in range(max_iter):
        p = schedule.order(r, prev)
        prev = p
        w = apply_fn(V[k], p)
        for j in range(k + 1):
            H[j, k] = V[j] @ w
            w = w - H[j, k] * V[j]
        H[k + 1, k] = np.linalg.norm(w)
        V.append(w / H[k + 1, k] if H[k + 1, k] > 0.0 else np.zeros_like(w))
        for j in range(k):
            H[j, k], H[j + 1, k] = (cs[j] * H[j, k] + sn[j] * H[j + 1, k],
                                    -sn[j] * H[j, k] + cs[j] * H[j + 1, k])
        den = math.hypot(H[k, k], H[k + 1, k])
        cs[k], sn[k] = H[k, k] / den, H[k + 1, k] / den
        H[k, k], H[k + 1, k] = den, 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        r = abs(g[k + 1]) / nb
        out.residuals.append(r)
        out.orders.append(p)
        if r < tol:
            out.converged = True
            break
    m = len(out.orders)
    y = np.linalg.solve(H[:m, :m], g[:m]) if m else np.zeros(0)
    out.x = sum((y[j] * V[j] for j in range(m)), np.zeros_like(b))
    return out
