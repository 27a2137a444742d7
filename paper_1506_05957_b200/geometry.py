"""Host-side panel geometry and quadrature rules (input preparation, O(P)).

The device path consumes Gauss points, weights, normals and areas produced
here.  They must be *bit-identical* to what the reference computes in
``pkg/src/fmmbem/quadrature.py:86-121`` because the octree replays the
reference's ``>`` comparisons against exact cell centres
(``octree.py:100-104``): on the mirror-symmetric icospheres many Gauss points
sit exactly on a split plane, and a one-ulp difference would move them to
the other octant (SURVEY.md finding 0.3).  So the arithmetic below uses the
same numpy primitives in the same order (mean / cross / norm / einsum).

Rules (published constants, ``quadrature.py:47-72``): the 4-point degree-3
rule with the centroid first, and the 19-point degree-9 rule.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np


def _cyc3(a):
    c = 1.0 - 2.0 * a
    return [(c, a, a), (a, c, a), (a, a, c)]


def _perm6(a, b):
    c = 1.0 - a - b
    return [(a, b, c), (a, c, b), (b, a, c), (b, c, a), (c, a, b), (c, b, a)]


def far_rule():
    """(bary (4,3), weights (4,)): centroid weight -27/48, three points at (0.6,0.2,0.2)."""
    bary = [(1 / 3, 1 / 3, 1 / 3)] + _cyc3(0.2)
    w = [-27 / 48] + [25 / 48] * 3
    return np.array(bary), np.array(w)


def near_rule():
    """(bary (19,3), weights (19,)): symmetric degree-9 rule."""
    bary = [(1 / 3, 1 / 3, 1 / 3)]
    w = [0.097135796282799]
    for a, wa in ((0.489682519198738, 0.031334700227139),
                  (0.437089591492937, 0.077827541004774),
                  (0.188203535619033, 0.079647738927210),
                  (0.044729513394453, 0.025577675658698)):
        bary += _cyc3(a)
        w += [wa] * 3
    bary += _perm6(0.741198598784498, 0.036838412054736)
    w += [0.043283539377289] * 6
    return np.array(bary), np.array(w)


FAR_BARY, FAR_W = far_rule()
NEAR_BARY, NEAR_W = near_rule()


def panel_geometry(pv: np.ndarray):
    """(centroid, unit normal, area) for panels pv (P, 3, 3); right-hand-rule normal."""
    v = np.asarray(pv, dtype=np.float64)
    cen = v.mean(axis=1)
    cr = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
    nrm = np.linalg.norm(cr, axis=1)
    if np.any(nrm == 0.0):
        raise ValueError("degenerate triangle")
    return cen, cr / nrm[:, None], 0.5 * nrm


def rule_points(pv: np.ndarray, bary: np.ndarray, w: np.ndarray):
    """Physical points (P, K, 3) and area-scaled weights (P, K) of a barycentric rule."""
    v = np.asarray(pv, dtype=np.float64)
    _, _, area = panel_geometry(v)
    pts = np.einsum("kc,pcd->pkd", bary, v)
    wts = area[:, None] * w[None, :]
    return pts, wts


@lru_cache(maxsize=8)
def gauss_legendre(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return np.ascontiguousarray(x), np.ascontiguousarray(w)


class PanelSet:
    """Everything the device operator needs about a mesh, in panel order.

    Attributes mirror ``BemOperator.__init__`` (``bemop.py:57-70``):
    ``centroids`` are the far rule's centroid point (bitwise the Gauss point 0
    so the self source drops out of every direct sum), ``src_pos``/``src_weight``
    the 4 Gauss points per panel flattened panel-major.
    """

    def __init__(self, mesh):
        pv = np.ascontiguousarray(mesh.panel_vertices, dtype=np.float64)
        self.panel_vertices = pv
        self.n_panels = int(pv.shape[0])
        _, self.normals, self.areas = panel_geometry(pv)
        pts, wts = rule_points(pv, FAR_BARY, FAR_W)
        self.centroids = np.ascontiguousarray(pts[:, 0])
        self.src_pos = np.ascontiguousarray(pts.reshape(-1, 3))
        self.src_weight = np.ascontiguousarray(wts.reshape(-1))
        fine_pts, fine_wts = rule_points(pv, NEAR_BARY, NEAR_W)
        self.fine_pos = np.ascontiguousarray(fine_pts)
        self.fine_weight = np.ascontiguousarray(fine_wts)
        self.normals = np.ascontiguousarray(self.normals)
        self.areas = np.ascontiguousarray(self.areas)
