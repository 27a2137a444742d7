"""Edge cases of the device path against the CPU oracle (oracle/fmm_oracle.py).

Single-leaf trees (no far field at all), a tree with one level of M2L, every
order below the rotation M2L threshold, zero right-hand sides, max_iter = 0,
non-contiguous inputs, and all three formulations at small sizes.  Bars as in
test_gpu_parity.py: mat-vec relative L2 <= 1e-10, GMRES iterations +-1,
solution <= 1e-6.
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-10


def _pair(mesh, formulation, n_crit, theta=0.5):
    from oracle import fmm_oracle as O
    from paper_1506_05957_b200.operator import GpuBemOperator

    op = GpuBemOperator(mesh, formulation, theta=theta, n_crit=n_crit)
    ref = O.OracleOperator(mesh, formulation, theta=theta, n_crit=n_crit)
    return op, ref


@pytest.mark.parametrize("formulation", ["laplace_first", "laplace_second", "stokes"])
def test_single_leaf_tree_is_pure_near_field(formulation):
    # 80 panels, n_crit above the point count: one leaf, no M2L pairs, every source near
    from paper_1506_05957_b200 import make_icosphere

    op, ref = _pair(make_icosphere(1), formulation, n_crit=1000)
    x = np.random.default_rng(3).uniform(-1.0, 1.0, op.shape[0])
    for p in (0, 3, 12):
        y, yr = op.apply(x, p), ref.apply(x, p)
        assert rel_l2(y, yr) <= MATVEC_TOL, (formulation, p, rel_l2(y, yr))


@pytest.mark.parametrize("p", [0, 1, 2, 3, 4, 5, 6])
def test_low_orders_around_the_rotation_threshold(p):
    # dense M2L below p = 3, rotation (DMMA) from p = 3
    from paper_1506_05957_b200 import make_icosphere

    op, ref = _pair(make_icosphere(2), "laplace_second", n_crit=16)
    x = np.random.default_rng(4).uniform(-1.0, 1.0, op.shape[0])
    y, yr = op.apply(x, p), ref.apply(x, p)
    assert rel_l2(y, yr) <= MATVEC_TOL, (p, rel_l2(y, yr))


def test_zero_rhs_and_zero_iterations():
    from paper_1506_05957_b200 import make_icosphere
    from paper_1506_05957_b200.solver import solve

    op, _ = _pair(make_icosphere(2), "laplace_second", n_crit=32)
    n = op.shape[0]
    res = solve(op, np.zeros(n), eta=1e-6, p_initial=8, p_min=3)
    assert res.converged and res.n_iterations == 0 and not np.any(res.x)
    b = np.random.default_rng(5).uniform(-1.0, 1.0, n)
    res0 = solve(op, b, eta=1e-6, p_initial=8, p_min=3, max_iter=0)
    assert res0.n_iterations == 0 and not res0.converged
    # a zero density maps to zero
    assert not np.any(op.apply(np.zeros(n), 8))


def test_non_contiguous_input_and_no_mutation():
    from paper_1506_05957_b200 import make_icosphere

    op, ref = _pair(make_icosphere(2), "laplace_second", n_crit=32)
    n = op.shape[0]
    big = np.random.default_rng(6).uniform(-1.0, 1.0, 2 * n)
    x = big[::2]  # strided view
    keep = x.copy()
    y = op.apply(x, 7)
    assert np.array_equal(x, keep)
    assert rel_l2(y, ref.apply(np.ascontiguousarray(x), 7)) <= MATVEC_TOL


@pytest.mark.parametrize("formulation", ["laplace_first", "laplace_second", "stokes"])
def test_small_relaxed_solves_match_the_oracle(formulation):
    from oracle import fmm_oracle as O
    from paper_1506_05957_b200 import make_icosphere
    from paper_1506_05957_b200.solver import solve

    op, ref = _pair(make_icosphere(2), formulation, n_crit=24)
    b = ref.apply(np.random.default_rng(7).uniform(-1.0, 1.0, op.shape[0]), 12)
    p0, pmin = (10, 5) if formulation == "stokes" else (10, 3)
    res = solve(op, b, eta=1e-6, p_initial=p0, p_min=pmin, relaxed=True)
    rr = O.gmres(ref.apply, b, O.RelaxationSchedule(p0, pmin, 1e-6, True), 1e-6, 100)
    assert abs(res.n_iterations - rr.n_iterations) <= 1
    assert rel_l2(res.x, rr.x) <= 1e-6


@pytest.mark.parametrize("theta", [0.3, 0.7])
def test_other_opening_angles(theta):
    from paper_1506_05957_b200 import make_icosphere

    op, ref = _pair(make_icosphere(2), "laplace_second", n_crit=16, theta=theta)
    x = np.random.default_rng(8).uniform(-1.0, 1.0, op.shape[0])
    for p in (4, 9):
        y, yr = op.apply(x, p), ref.apply(x, p)
        assert rel_l2(y, yr) <= MATVEC_TOL, (theta, p, rel_l2(y, yr))


@pytest.mark.parametrize("formulation", ["laplace_second", "stokes"])
def test_deep_tree_n_crit_1(formulation):
    # one point per leaf where possible: deep trees, long root paths, many tiny P2P items
    from paper_1506_05957_b200 import make_icosphere

    op, ref = _pair(make_icosphere(1), formulation, n_crit=1)
    x = np.random.default_rng(9).uniform(-1.0, 1.0, op.shape[0])
    for p in (3, 10):
        y, yr = op.apply(x, p), ref.apply(x, p)
        assert rel_l2(y, yr) <= MATVEC_TOL, (formulation, p, rel_l2(y, yr))


def test_double_layer_far_from_the_origin():
    # 8 rotated red-blood-cell surfaces on a 2x2x2 lattice (|x| up to ~13 um, level-3 cells):
    # the expanded-form near field centres on the target leaf, so its cancellation does not
    # grow with the distance to the origin
    from paper_1506_05957_b200 import make_rbc_lattice

    op, ref = _pair(make_rbc_lattice(2, level=3), "laplace_second", n_crit=64)
    x = np.random.default_rng(10).uniform(-1.0, 1.0, op.shape[0])
    for p in (5, 12):
        y, yr = op.apply(x, p), ref.apply(x, p)
        assert rel_l2(y, yr) <= MATVEC_TOL, (p, rel_l2(y, yr))


@pytest.mark.parametrize("n_crit", [300, 700])
def test_fewer_near_field_items_than_ctas(n_crit):
    # a handful of large leaves: the persistent near field has fewer work items than CTAs
    # (idle CTAs take the empty-schedule path of the stage hand-off), items near the source cap
    from paper_1506_05957_b200 import make_icosphere

    op, ref = _pair(make_icosphere(3), "laplace_second", n_crit=n_crit)
    x = np.random.default_rng(11).uniform(-1.0, 1.0, op.shape[0])
    for p in (3, 9):
        y, yr = op.apply(x, p), ref.apply(x, p)
        assert rel_l2(y, yr) <= MATVEC_TOL, (n_crit, p, rel_l2(y, yr))
