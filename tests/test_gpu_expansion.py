"""Single-expansion API on the device (fmm.py:29-81, 488-493) against the reference.

Coefficients and values are compared with tests/golden/expansion.npz, written by the
unmodified reference (tools/make_goldens_expansion.py); the reference's own unit properties
(test_harmonics.py: M2M and L2L exactness, M2L / P2M convergence, gradients vs finite
differences; acceptance criterion 7's cluster bound) are re-run on the device operators.
"""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

ORDERS = (0, 1, 3, 8, 14, 20)


def _close(a, b, rtol=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(np.max(np.abs(b)), 1e-300)
    return np.max(np.abs(a - b)) <= rtol * scale


@pytest.mark.parametrize("p", ORDERS)
def test_operators_match_reference_goldens(p):
    from paper_1506_05957_b200 import fmm

    g = load_golden("expansion")
    src, q, q2, nrm = g["src"], g["q"], g["q2"], g["nrm"]
    e = fmm.p2m(src, q, np.zeros(3), p)
    assert e.coeffs.shape == ((p + 1) ** 2,)
    assert _close(e.coeffs, g[f"p2m_q_p{p}"])
    ed = fmm.p2m(src, np.zeros(len(src)), np.zeros(3), p, dipoles=q[:, None] * nrm)
    assert _close(ed.coeffs, g[f"p2m_d_p{p}"])
    e2 = fmm.p2m(src, q2, np.array([0.1, -0.05, 0.02]), p)
    assert e2.coeffs.shape == (2, (p + 1) ** 2) and _close(e2.coeffs, g[f"p2m_q2_p{p}"])
    pot, grad = fmm.m2p(e, g["tgt_far"], want_gradient=True)
    assert _close(pot, g[f"m2p_p{p}"]) and _close(grad, g[f"m2p_grad_p{p}"])
    assert _close(fmm.m2m(e, np.array([0.3, -0.2, 0.1])).coeffs, g[f"m2m_p{p}"])
    loc = fmm.m2l(e, np.array([3.0, 0.0, 0.0]))
    assert _close(loc.coeffs, g[f"m2l_p{p}"])
    assert _close(fmm.l2l(loc, np.array([3.1, 0.05, -0.1])).coeffs, g[f"l2l_p{p}"])
    pot, grad = fmm.l2p(loc, g["tgt_loc"], want_gradient=True)
    assert _close(pot, g[f"l2p_p{p}"]) and _close(grad, g[f"l2p_grad_p{p}"])


def test_scalar_helpers_match_reference():
    from paper_1506_05957_b200 import fmm

    g = load_golden("expansion")
    assert [fmm.required_p(e) for e in (1.0, 0.5, 1e-3, 0.5 ** 12, 1e-10)] == list(g["required_p"])
    assert np.allclose([fmm.multipole_error_bound(3.0, 0.5, 1.0, p) for p in (2, 5, 8)],
                       g["error_bound"], rtol=1e-15)
    with pytest.raises(ValueError):
        fmm.required_p(0.0)
    with pytest.raises(ValueError):
        fmm.multipole_error_bound(1.0, 1.0, 0.5, 4)
    with pytest.raises(ValueError):
        fmm.Expansion(np.zeros(3), 3, np.zeros(15))
    with pytest.raises(ValueError):
        fmm.p2m(np.zeros((2, 3)) + 1.0, np.ones(2), np.zeros(3), 21)


def _cluster(rng, n=40, radius=0.5):
    v = rng.normal(size=(n, 3))
    v *= radius * rng.uniform(0.2, 1.0, size=(n, 1)) / np.linalg.norm(v, axis=1, keepdims=True)
    return v


def _direct(src, q, tgt):
    r = np.linalg.norm(tgt[:, None, :] - src[None, :, :], axis=-1)
    return (q[None, :] / r).sum(axis=1) / (4 * np.pi)


def test_reference_unit_properties_on_device():
    # test_harmonics.py:19-66 and acceptance criterion 7 (test_acceptance.py:250-260)
    from paper_1506_05957_b200 import fmm

    rng = np.random.default_rng(7)
    src = _cluster(rng)
    q = rng.uniform(-1.0, 1.0, size=len(src))
    tgt = np.array([[2.0, 0.3, -0.4], [0.0, -2.5, 1.0]])
    ref = _direct(src, q, tgt)
    errs = [np.max(np.abs(fmm.m2p(fmm.p2m(src, q, np.zeros(3), p), tgt) / (4 * np.pi) - ref) / np.abs(ref))
            for p in (4, 8, 12)]
    assert errs[0] < 1e-2 and errs[1] < errs[0] / 10 and errs[2] < 1e-8
    shifted = np.array([0.3, -0.2, 0.1])
    np.testing.assert_allclose(fmm.m2m(fmm.p2m(src, q, np.zeros(3), 8), shifted).coeffs,
                               fmm.p2m(src, q, shifted, 8).coeffs, atol=1e-12)
    local = fmm.m2l(fmm.p2m(src, q, np.zeros(3), 8), np.array([3.0, 0.0, 0.0]))
    moved = fmm.l2l(local, np.array([3.1, 0.05, -0.1]))
    t = np.array([[3.15, 0.1, -0.05]])
    np.testing.assert_allclose(fmm.l2p(moved, t), fmm.l2p(local, t), rtol=1e-12)
    for which in ("multipole", "local"):
        exp = fmm.p2m(src, q, np.zeros(3), 10)
        if which == "local":
            exp = fmm.m2l(exp, np.array([2.5, 0.1, 0.0]))
            ev, t = fmm.l2p, np.array([[2.6, 0.2, -0.1]])
        else:
            ev, t = fmm.m2p, np.array([[2.0, 0.4, -0.3]])
        _, grad = ev(exp, t, want_gradient=True)
        for axis in range(3):
            step = np.zeros(3)
            step[axis] = 1e-6
            fd = (ev(exp, t + step)[0] - ev(exp, t - step)[0]) / 2e-6
            assert abs(grad[0, axis] - fd) < 1e-6 * max(1.0, abs(fd))
    a = 0.5
    rng = np.random.default_rng(0)
    c = rng.normal(size=(200, 3))
    c *= a * rng.uniform(0.1, 1.0, size=(200, 1)) / np.linalg.norm(c, axis=1, keepdims=True)
    qc = rng.uniform(0.0, 1.0, size=200)
    t = np.array([[2 * a, 0.0, 0.0]])
    exact = _direct(c, qc, t)[0]
    for p in (2, 5, 8):
        approx = fmm.m2p(fmm.p2m(c, qc, np.zeros(3), p), t)[0] / (4 * np.pi)
        assert abs(approx - exact) <= fmm.multipole_error_bound(qc.sum(), a, 2 * a, p) / (4 * np.pi)
