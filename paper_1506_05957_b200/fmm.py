"""N-body evaluation through the device FMM (reference ``fmm.evaluate``, fmm.py:456-485),
and the reference's single-expansion API (``Expansion``, ``p2m``, ``m2m``, ``m2l``, ``l2l``,
``m2p``, ``l2p``, ``required_p``, ``multipole_error_bound``; fmm.py:29-81, 488-493) with the
operators on the device (``fmmbem_expansion_*``, csrc/expansion_api.cu).

``evaluate(kernel, src_pos, weights, targets, p, ...)`` returns the FMM approximation of
the reference's ``kernels.direct_sum`` for the four kernels, with the same channel
decompositions: Laplace single layer (charges), double layer (dipoles w n), stokeslet
(four charge channels [f, y.f] with gradients, fmm.py:422-433) and stresslet (seven dipole
channels with gradients, fmm.py:436-453).  Far and near fields are computed in one device
call (``GpuFmmPlan`` parts = far + near).  Only ``policy="fmm"`` is served.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .operator import GpuFmmPlan

FOUR_PI = 4.0 * np.pi


class KernelKind(enum.Enum):
    """Reference ``kernels.KernelKind`` (kernels.py:15-19)."""
    LAPLACE_SINGLE = "laplace_single"
    LAPLACE_DOUBLE = "laplace_double"
    STOKESLET = "stokeslet"
    STRESSLET = "stresslet"


def stokeslet_channels(src_pos, strengths):
    """(4, Ns) charges: f_x, f_y, f_z and y.f (fmm.py:422-425)."""
    f = np.asarray(strengths, dtype=float)
    return np.vstack([f.T, np.einsum("si,si->s", np.asarray(src_pos, dtype=float), f)])


def combine_stokeslet(targets, pot, grad):
    """u_i = phi_i - x_c d_i phi_c + d_i psi (fmm.py:428-433)."""
    u = pot[:3].T.copy()
    u -= np.einsum("tc,cti->ti", np.asarray(targets, dtype=float), grad[:3])
    u += grad[3]
    return u


def stresslet_channels(src_pos, strengths, normals):
    """(7, Ns, 3) dipoles: Phi_c = f_c n, Lambda_c = n_c f, Psi = (y.f) n (fmm.py:436-445)."""
    f = np.asarray(strengths, dtype=float)
    n = np.asarray(normals, dtype=float)
    dip = np.empty((7, len(f), 3))
    for c in range(3):
        dip[c] = f[:, c:c + 1] * n
        dip[3 + c] = n[:, c:c + 1] * f
    dip[6] = np.einsum("si,si->s", np.asarray(src_pos, dtype=float), f)[:, None] * n
    return dip


def combine_stresslet(targets, pot, grad):
    """u_i = 2 Lambda_i - 2 x_c d_i Phi_c + 2 d_i Psi (fmm.py:448-453)."""
    u = 2.0 * pot[3:6].T.copy()
    u -= 2.0 * np.einsum("tc,cti->ti", np.asarray(targets, dtype=float), grad[:3])
    u += 2.0 * grad[6]
    return u


def evaluate(kernel, src_pos, weights, targets, p, theta=0.5, n_crit=126, normals=None,
             policy="fmm", plan=None):
    """FMM approximation of ``kernels.direct_sum`` (fmm.py:456-485); a prebuilt
    :class:`GpuFmmPlan` for the same geometry amortises the tree construction."""
    kind = KernelKind(kernel)
    src_pos = np.atleast_2d(np.asarray(src_pos, dtype=float))
    targets = np.atleast_2d(np.asarray(targets, dtype=float))
    if plan is None:
        plan = GpuFmmPlan(src_pos, targets, n_crit=n_crit, theta=theta, policy=policy)
    both = 3  # far field + near field in one device call
    if kind is KernelKind.LAPLACE_SINGLE:
        q = np.asarray(weights, dtype=float)
        return plan._evaluate(q, None, p, False, both) / FOUR_PI
    if kind is KernelKind.LAPLACE_DOUBLE:
        if normals is None:
            raise ValueError("the double layer needs source normals")
        dip = np.asarray(weights, dtype=float)[:, None] * np.asarray(normals, dtype=float)
        return plan._evaluate(None, dip, p, False, both) / FOUR_PI
    if kind is KernelKind.STOKESLET:
        pot, grad = plan._evaluate(stokeslet_channels(src_pos, weights), None, p, True, both)
        return combine_stokeslet(targets, pot, grad)
    if normals is None:
        raise ValueError("the stresslet needs source normals")
    pot, grad = plan._evaluate(None, stresslet_channels(src_pos, weights, normals), p, True, both)
    return combine_stresslet(targets, pot, grad)


# ---------------------------------------------------------------- single expansions
def num_coeffs(p):
    """(p+1)^2 (harmonics.py:30-31)."""
    return (p + 1) ** 2


def required_p(eps):
    """Expansion order for accuracy eps at separation ratio 2 (fmm.py:29-33)."""
    if not 0.0 < eps <= 1.0:
        raise ValueError("eps must be in (0, 1]")
    return max(0, math.ceil(-math.log2(eps)))


def multipole_error_bound(total_abs_charge, cluster_radius, distance, p):
    """Greengard-style truncation bound sum|q| / (r - a) (a/r)^(p+1) (fmm.py:488-493)."""
    a, r = cluster_radius, distance
    if r <= a:
        raise ValueError("target must lie outside the cluster radius")
    return total_abs_charge / (r - a) * (a / r) ** (p + 1)


@dataclass
class Expansion:
    """Truncated multipole or local coefficient set about a center (fmm.py:36-49).
    ``coeffs`` (..., (p+1)^2) complex in the reference's flat layout n^2 + n + m."""

    center: np.ndarray
    order: int
    coeffs: np.ndarray

    def __post_init__(self):
        self.center = np.asarray(self.center, dtype=float)
        self.coeffs = np.asarray(self.coeffs, dtype=complex)
        if self.coeffs.shape[-1] != num_coeffs(self.order):
            raise ValueError("coefficient count must be (p+1)^2")


def _device():
    try:
        import torch

        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def _check_p(p):
    if not 0 <= int(p) <= 20:
        raise ValueError("expansion order p must be in [0, 20]")
    return int(p)


def p2m(src_pos, charges, center, p, dipoles=None):
    """Multipole of point charges (+ dipoles) about ``center`` (fmm.py:52-54,
    harmonics.particle_to_multipole :221-235); leading axes of charges/dipoles are channels."""
    p = _check_p(p)
    rel = np.ascontiguousarray(np.atleast_2d(np.asarray(src_pos, dtype=float)) -
                               np.asarray(center, dtype=float))
    n = rel.shape[0]
    q = None if charges is None else np.asarray(charges, dtype=float)
    d = None if dipoles is None else np.asarray(dipoles, dtype=float)
    lead = q.shape[:-1] if q is not None else d.shape[:-2]
    C = int(np.prod(lead)) if lead else 1
    qq = None if q is None else N.f64(np.broadcast_to(q, lead + (n,)).reshape(C, n))
    dd = None if d is None else N.f64(np.broadcast_to(d, lead + (n, 3)).reshape(C, n, 3))
    out = np.empty((C, num_coeffs(p)), dtype=complex)
    N.check(N.load().fmmbem_expansion_p2m(N.dptr(rel), n, None if qq is None else N.dptr(qq),
                                          None if dd is None else N.dptr(dd), C, p,
                                          out.ctypes.data_as(N._c_double_p), _device()))
    return Expansion(center, p, out.reshape(lead + (num_coeffs(p),)))


def _translate(kind, expansion, d, new_center):
    p = _check_p(expansion.order)
    c = np.ascontiguousarray(expansion.coeffs, dtype=complex)
    lead = c.shape[:-1]
    C = int(np.prod(lead)) if lead else 1
    out = np.empty((C, num_coeffs(p)), dtype=complex)
    dv = N.f64(np.asarray(d, dtype=float).reshape(3))
    N.check(N.load().fmmbem_expansion_translate(kind, N.dptr(dv), C, p,
                                                c.reshape(C, -1).ctypes.data_as(N._c_double_p),
                                                out.ctypes.data_as(N._c_double_p), _device()))
    return Expansion(new_center, p, out.reshape(lead + (num_coeffs(p),)))


def m2m(expansion, new_center):
    """Shift a multipole to ``new_center`` (fmm.py:56-59; exact)."""
    return _translate(0, expansion, expansion.center - np.asarray(new_center, dtype=float), new_center)


def m2l(expansion, target_center):
    """Multipole to local about ``target_center`` (fmm.py:62-65)."""
    return _translate(1, expansion, np.asarray(target_center, dtype=float) - expansion.center,
                      target_center)


def l2l(expansion, new_center):
    """Shift a local expansion to ``new_center`` (fmm.py:68-71; exact)."""
    return _translate(2, expansion, np.asarray(new_center, dtype=float) - expansion.center, new_center)


def _evaluate_expansion(kind, expansion, targets, want_gradient):
    p = _check_p(expansion.order)
    rel = np.ascontiguousarray(np.atleast_2d(np.asarray(targets, dtype=float)) - expansion.center)
    c = np.ascontiguousarray(expansion.coeffs, dtype=complex)
    single = c.ndim == 1
    c2 = c.reshape(-1, num_coeffs(p))
    C, n = c2.shape[0], rel.shape[0]
    pot = np.empty((C, n))
    grad = np.empty((C, n, 3)) if want_gradient else None
    N.check(N.load().fmmbem_expansion_evaluate(kind, c2.ctypes.data_as(N._c_double_p), C, p,
                                               N.dptr(rel), n, 1 if want_gradient else 0,
                                               N.dptr(pot), None if grad is None else N.dptr(grad),
                                               _device()))
    if single:
        return (pot[0], grad[0]) if want_gradient else pot[0]
    return (pot, grad) if want_gradient else pot


def m2p(expansion, targets, want_gradient=False):
    """Evaluate a multipole at targets (fmm.py:74-76, harmonics.multipole_to_point)."""
    return _evaluate_expansion(0, expansion, targets, want_gradient)


def l2p(expansion, targets, want_gradient=False):
    """Evaluate a local expansion at targets (fmm.py:79-81, harmonics.local_to_point)."""
    return _evaluate_expansion(1, expansion, targets, want_gradient)
