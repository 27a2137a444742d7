"""CPU: the relaxation schedule (solver.py:20-47 of the reference) and its device twin.

The device GMRES applies the same rules in C++ (csrc/gmres.cu); the GPU tests
check the resulting order histories against the reference's goldens.
"""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import fmm_oracle as O
from paper_1506_05957_b200.solver import RelaxationSchedule, SolveResult, relax_eps, schedule_p


@given(st.floats(1e-14, 10.0), st.floats(1e-12, 0.5))
@settings(max_examples=200, deadline=None)
def test_relax_eps_in_unit_interval(r, eta):
    e = relax_eps(r, eta)
    assert 0.0 < e <= 1.0
    assert e >= eta - 1e-300


@given(st.floats(1e-14, 10.0), st.floats(1e-12, 0.5), st.integers(1, 20), st.integers(0, 20))
@settings(max_examples=200, deadline=None)
def test_schedule_p_clamped(r, eta, p_initial, p_min):
    p_min = min(p_min, p_initial)
    p = schedule_p(r, eta, p_initial, p_min)
    assert p_min <= p <= p_initial


def test_schedule_p_monotone_in_residual():
    ps = [schedule_p(r, 1e-6, 12, 3) for r in np.logspace(0, -7, 50)]
    assert all(a >= b for a, b in zip(ps, ps[1:]))


def test_first_iteration_uses_p_initial():
    assert RelaxationSchedule(12, 3, 1e-6, True).order(1.0, 12) == 12
    assert RelaxationSchedule(12, 3, 1e-6, False).order(1e-3, 4) == 12


@given(st.floats(1e-9, 1.0), st.integers(1, 20))
@settings(max_examples=100, deadline=None)
def test_matches_oracle_restatement(r, prev):
    a = RelaxationSchedule(14, 3, 1e-6, True).order(r, prev)
    b = O.RelaxationSchedule(14, 3, 1e-6, True).order(r, prev)
    assert a == b


def test_rejects_bad_eta():
    with pytest.raises(ValueError):
        relax_eps(0.5, 0.0)


def test_save_history(tmp_path):
    res = SolveResult(x=np.zeros(2), residuals=[0.5, 1e-7], orders=[12, 5], converged=True)
    path = tmp_path / "h.csv"
    res.save_history(path)
    lines = path.read_text().splitlines()
    assert lines[0] == "iteration,residual,p"
    assert lines[2].split(",")[2] == "5"
    assert math.isclose(float(lines[1].split(",")[1]), 0.5)


def test_oracle_gmres_solves_dense_system():
    """GMRES semantics (solver.py:69-134) on a small well-conditioned dense system."""
    rng = np.random.default_rng(0)
    A = np.eye(30) * 4 + rng.uniform(-0.5, 0.5, (30, 30))
    b = rng.uniform(-1, 1, 30)
    r = O.gmres(lambda x, p: A @ x, b, O.RelaxationSchedule(5, 1, 1e-12, False), 1e-12, 60)
    assert r.converged
    np.testing.assert_allclose(r.x, np.linalg.solve(A, b), rtol=1e-9)
    assert all(a >= b for a, b in zip(r.residuals, r.residuals[1:]))
