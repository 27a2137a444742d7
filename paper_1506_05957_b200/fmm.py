"""N-body evaluation through the device FMM (reference ``fmm.evaluate``, fmm.py:456-485).

``evaluate(kernel, src_pos, weights, targets, p, ...)`` returns the FMM approximation of
the reference's ``kernels.direct_sum`` for the four kernels, with the same channel
decompositions: Laplace single layer (charges), double layer (dipoles w n), stokeslet
(four charge channels [f, y.f] with gradients, fmm.py:422-433) and stresslet (seven dipole
channels with gradients, fmm.py:436-453).  Far and near fields are computed in one device
call (``GpuFmmPlan`` parts = far + near).  Only ``policy="fmm"`` is served.
"""

from __future__ import annotations

import enum

import numpy as np

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
