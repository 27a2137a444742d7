"""fmm.evaluate on the device (reference fmm.py:456-485) against the oracle's far + near
fields composed the reference's way (oracle/fmm_oracle.py OraclePlan), and run_scaling."""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

FOUR_PI = 4.0 * np.pi


def _points(n, seed):
    rng = np.random.default_rng(seed)
    src = rng.uniform(-1.0, 1.0, (n, 3))
    tgt = rng.uniform(-1.0, 1.0, (n // 2, 3))
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1)[:, None]
    return rng, src, tgt, nrm


@pytest.mark.parametrize("kind", ["laplace_single", "laplace_double", "stokeslet", "stresslet"])
def test_evaluate_matches_the_oracle(kind):
    from oracle import fmm_oracle as O
    from paper_1506_05957_b200 import fmm

    rng, src, tgt, nrm = _points(1500, 3)
    p, n_crit = 7, 40
    w = rng.uniform(-1.0, 1.0, len(src)) if kind.startswith("laplace") else rng.uniform(-1.0, 1.0, (len(src), 3))
    got = fmm.evaluate(kind, src, w, tgt, p=p, n_crit=n_crit, normals=nrm)
    plan = O.OraclePlan(src, tgt, n_crit=n_crit, theta=0.5)
    if kind == "laplace_single":
        want = (plan.far_field(charges=w, p=p) + plan.near_field(charges=w)) / FOUR_PI
    elif kind == "laplace_double":
        d = w[:, None] * nrm
        want = (plan.far_field(dipoles=d, p=p) + plan.near_field(dipoles=d)) / FOUR_PI
    elif kind == "stokeslet":
        q = fmm.stokeslet_channels(src, w)
        pot, grad = plan.far_field(charges=q, p=p, want_gradient=True)
        npot, ngrad = plan.near_field(charges=q, want_gradient=True)
        want = fmm.combine_stokeslet(tgt, pot + npot, grad + ngrad)
    else:
        d = fmm.stresslet_channels(src, w, nrm)
        pot, grad = plan.far_field(dipoles=d, p=p, want_gradient=True)
        npot, ngrad = plan.near_field(dipoles=d, want_gradient=True)
        want = fmm.combine_stresslet(tgt, pot + npot, grad + ngrad)
    assert got.shape == want.shape
    assert rel_l2(got.ravel(), want.ravel()) <= 1e-10


def test_evaluate_converges_to_the_direct_sum():
    from paper_1506_05957_b200 import fmm

    rng, src, tgt, _ = _points(2000, 4)
    q = rng.uniform(-1.0, 1.0, len(src))
    r = np.linalg.norm(tgt[:, None, :] - src[None, :, :], axis=2)
    direct = (q[None, :] / r).sum(axis=1) / FOUR_PI
    ps = (2, 6, 12)
    errs = [rel_l2(fmm.evaluate("laplace_single", src, q, tgt, p=p, n_crit=64), direct) for p in ps]
    assert errs[0] > errs[1] > errs[2], errs
    # the reference's accuracy bound at theta = 0.5 (test_fmm.py:61-68): error <= 2^-p
    assert all(e <= 2.0 ** -p for e, p in zip(errs, ps)), errs


def test_run_scaling_reports_a_slope():
    from paper_1506_05957_b200.study import run_scaling

    rep = run_scaling([20000, 40000, 80000], p=5, n_crit=126, repeats=2)
    assert [r["N"] for r in rep.records] == [20000, 40000, 80000]
    assert all(r["time"] > 0 for r in rep.records)
    assert np.isfinite(rep.derived["slope"])
