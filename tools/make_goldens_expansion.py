"""Golden vectors of the reference's single-expansion API (fmm.py:29-81, 488-493), made by
the UNMODIFIED reference in this container.

Usage: PYTHONPATH=/root/reference/pkg/src:. python tools/make_goldens_expansion.py
Writes tests/golden/expansion.npz: seeded clusters / targets, p2m (charges, dipoles, 2
channels), m2m, m2l, l2l coefficient vectors, m2p / l2p values and gradients, required_p and
multipole_error_bound values.  Coefficients in the reference's flat layout n^2 + n + m.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from tools.make_goldens import OUT  # noqa: E402


def main():
    from fmmbem import fmm

    rng = np.random.default_rng(11)
    src = rng.normal(size=(40, 3))
    src *= 0.5 * rng.uniform(0.2, 1.0, size=(40, 1)) / np.linalg.norm(src, axis=1, keepdims=True)
    q = rng.uniform(-1.0, 1.0, size=40)
    q2 = rng.uniform(-1.0, 1.0, size=(2, 40))
    nrm = rng.normal(size=(40, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    tgt_far = np.array([[2.0, 0.3, -0.4], [0.0, -2.5, 1.0], [-1.7, 1.1, 0.9]])
    tgt_loc = np.array([[3.15, 0.1, -0.05], [2.9, 0.2, -0.1], [3.1, -0.2, 0.15]])
    out = {"src": src, "q": q, "q2": q2, "nrm": nrm, "tgt_far": tgt_far, "tgt_loc": tgt_loc}
    for p in (0, 1, 3, 8, 14, 20):
        e = fmm.p2m(src, q, np.zeros(3), p)
        out[f"p2m_q_p{p}"] = e.coeffs
        out[f"m2p_p{p}"], out[f"m2p_grad_p{p}"] = fmm.m2p(e, tgt_far, want_gradient=True)
        ed = fmm.p2m(src, np.zeros(40), np.zeros(3), p, dipoles=q[:, None] * nrm)
        out[f"p2m_d_p{p}"] = ed.coeffs
        out[f"p2m_q2_p{p}"] = fmm.p2m(src, q2, np.array([0.1, -0.05, 0.02]), p).coeffs
        out[f"m2m_p{p}"] = fmm.m2m(e, np.array([0.3, -0.2, 0.1])).coeffs
        loc = fmm.m2l(e, np.array([3.0, 0.0, 0.0]))
        out[f"m2l_p{p}"] = loc.coeffs
        out[f"l2l_p{p}"] = fmm.l2l(loc, np.array([3.1, 0.05, -0.1])).coeffs
        out[f"l2p_p{p}"], out[f"l2p_grad_p{p}"] = fmm.l2p(loc, tgt_loc, want_gradient=True)
    out["required_p"] = np.array([fmm.required_p(e) for e in (1.0, 0.5, 1e-3, 0.5 ** 12, 1e-10)])
    out["error_bound"] = np.array([fmm.multipole_error_bound(3.0, 0.5, 1.0, p) for p in (2, 5, 8)])
    np.savez_compressed(os.path.join(OUT, "expansion.npz"), **out)
    print("wrote expansion.npz")


if __name__ == "__main__":
    main()
