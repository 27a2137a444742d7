"""Study harness (paper_1506_05957_b200/study.py).

CPU: the report format and the refinement-triple formulas (reference
`study.py:21-92`) on known answers.  GPU: the relaxed-vs-fixed comparison and a
convergence sequence on small spheres through the device path.
"""

import math

import numpy as np
import pytest

from paper_1506_05957_b200.study import StudyReport, observed_order, richardson


def test_refinement_triple_known_answers():
    # f_i = 1 + 4^(-2 i): order 2 at refinement ratio 4, limit 1
    f = [1.0 + 4.0 ** (-2 * i) for i in range(3)]
    assert math.isclose(observed_order(*f, c=4.0), 2.0, rel_tol=1e-12)
    assert math.isclose(richardson(*f), 1.0, rel_tol=1e-12)
    with pytest.raises(ValueError):
        observed_order(1.0, 2.0, 1.5)  # not monotone
    with pytest.raises(ValueError):
        observed_order(*f, c=1.0)
    with pytest.raises(ValueError):
        richardson(1.0, 2.0, 3.0)  # linear: degenerate


def test_report_round_trip(tmp_path):
    rep = StudyReport("relaxation", {"problem": "laplace2", "ncrit_candidates": [16, 64]})
    rep.records += [{"n_crit": 16, "relaxed": True, "time": 0.25},
                    {"n_crit": 64, "relaxed": False, "time": 0.5, "iterations": 9}]
    rep.derived["speedup"] = 2.0
    path = tmp_path / "r.txt"
    rep.write(path)
    back = StudyReport.read(path)
    assert back.kind == rep.kind and back.params == rep.params
    assert back.records == rep.records and back.derived == rep.derived
    rep.write_csv(tmp_path / "r.csv")
    lines = (tmp_path / "r.csv").read_text().splitlines()
    assert lines[0] == "n_crit,relaxed,time,iterations" and len(lines) == 3


@pytest.mark.gpu
def test_relaxation_comparison_on_device():
    from paper_1506_05957_b200.study import run_relaxation_comparison

    rep = run_relaxation_comparison("laplace2", level=3, tol=1e-6, p_initial=10, p_min=3,
                                    ncrit_candidates=(16, 64), repeats=1, max_iter=60)
    assert len(rep.records) == 4 and all(r["converged"] for r in rep.records)
    assert {r["n_crit"] for r in rep.records} == {16, 64}
    d = rep.derived
    assert d["speedup"] > 0 and d["best_ncrit_relaxed"] in (16, 64)
    # relaxation changes the far-field accuracy, not the converged answer
    assert d["solution_difference"] < 1e-4
    assert abs(d["iterations_relaxed"] - d["iterations_fixed"]) <= 3


@pytest.mark.gpu
def test_convergence_sequence_on_device():
    from paper_1506_05957_b200.study import run_convergence

    rep = run_convergence("laplace2", levels=[1, 2, 3], p=10, tol=1e-8, n_crit=32, p_min=3)
    err = [r["error"] for r in rep.records]
    assert all(r["converged"] for r in rep.records)
    assert err[0] > err[1] > err[2]
    assert np.isfinite(rep.derived["order"]) and rep.derived["order"] > 0.5


def _study_golden():
    import json

    from conftest import load_golden

    g = load_golden("study")
    return g, json


@pytest.mark.gpu
@pytest.mark.parametrize("problem,kw", [
    ("laplace2", dict(level=3, tol=1e-6, p_initial=10, p_min=3, ncrit_candidates=(16, 64))),
    ("stokes", dict(level=2, tol=1e-5, p_initial=12, p_min=5, ncrit_candidates=(16, 64)))])
def test_relaxation_comparison_matches_the_reference(problem, kw):
    """Same records as the reference's run_relaxation_comparison (study.py:207-242, run by
    tools/make_goldens_study.py): per (n_crit, relaxed) the panel count, the iteration count
    (+-1) and convergence; wall times are machine properties and are not compared."""
    from paper_1506_05957_b200.study import run_relaxation_comparison

    g, json = _study_golden()
    want = json.loads(str(g[f"relax_{problem}_records"]))
    rep = run_relaxation_comparison(problem, repeats=1, warmup=0, **kw)
    got = [{k: r[k] for k in ("N", "n_crit", "relaxed", "iterations", "converged")} for r in rep.records]
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert (a["N"], a["n_crit"], a["relaxed"], a["converged"]) == \
               (b["N"], b["n_crit"], b["relaxed"], b["converged"])
        assert abs(a["iterations"] - b["iterations"]) <= 1, (a, b)


@pytest.mark.gpu
def test_convergence_study_matches_the_reference():
    """run_convergence (study.py:143-191) on the same refinement sequence: panel counts,
    iterations and orders equal, errors to 1e-6 relative, the observed order to 1e-5."""
    from paper_1506_05957_b200.study import run_convergence

    g, json = _study_golden()
    want = json.loads(str(g["conv_laplace2_records"]))
    rep = run_convergence("laplace2", levels=[1, 2, 3], p=10, tol=1e-8, n_crit=32, p_min=3)
    for a, b in zip(rep.records, want):
        assert (a["N"], a["iterations"], list(a["orders"])) == (b["N"], b["iterations"], b["orders"])
        assert abs(a["error"] - b["error"]) <= 1e-6 * b["error"]
    assert abs(rep.derived["order"] - float(g["conv_laplace2_order"])) <= 1e-5
