"""Drop-in semantics of the solver/operator API against the reference's (solver.py:69-143).

* callback(k, residual, p) fires after EVERY iteration, inside the solve (solver.py:122-123),
  and an exception it raises propagates out of gmres().
* schedule.eta drives the order and tol the stop test independently (solver.py:41-47, :124).
* gmres() accepts any callable apply_fn (the reference loop around it).
* fmmbem_op_apply_device is ordered on the caller's CUDA stream.
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _ops(formulation="laplace_second", level=2, n_crit=32):
    from oracle import fmm_oracle as O
    from paper_1506_05957_b200 import make_icosphere
    from paper_1506_05957_b200.operator import GpuBemOperator

    mesh = make_icosphere(level)
    return (GpuBemOperator(mesh, formulation, theta=0.5, n_crit=n_crit),
            O.OracleOperator(mesh, formulation, theta=0.5, n_crit=n_crit))


def test_callback_fires_per_iteration_during_the_solve():
    from paper_1506_05957_b200.solver import RelaxationSchedule, gmres

    op, ref = _ops("laplace_first")
    b = ref.apply(np.ones(op.shape[0]), 12)
    seen = []
    res = gmres(op.apply, b, RelaxationSchedule(10, 3, 1e-6, True), tol=1e-6, max_iter=50,
                callback=lambda k, r, p: seen.append((k, r, p)))
    assert [s[0] for s in seen] == list(range(1, res.n_iterations + 1))
    assert [s[1] for s in seen] == res.residuals and [s[2] for s in seen] == res.orders


def test_callback_exception_stops_and_propagates():
    from paper_1506_05957_b200.solver import RelaxationSchedule, gmres

    op, ref = _ops("laplace_first")
    b = ref.apply(np.ones(op.shape[0]), 12)
    calls = []

    def cb(k, r, p):
        calls.append(k)
        if k == 2:
            raise KeyError("stop here")

    with pytest.raises(KeyError):
        gmres(op.apply, b, RelaxationSchedule(10, 3, 1e-8, True), tol=1e-8, max_iter=50, callback=cb)
    assert calls == [1, 2]


def test_eta_and_tol_are_independent():
    # a coarse eta relaxes p much earlier than tol would; orders and iterations follow the oracle
    from oracle import fmm_oracle as O
    from paper_1506_05957_b200.solver import RelaxationSchedule, gmres

    op, ref = _ops("laplace_first")
    b = ref.apply(np.ones(op.shape[0]), 12)
    res = gmres(op.apply, b, RelaxationSchedule(12, 2, 1e-3, True), tol=1e-9, max_iter=60)
    sched = O.RelaxationSchedule()
    sched.p_initial, sched.p_min, sched.eta, sched.relaxed = 12, 2, 1e-3, True
    rr = O.gmres(ref.apply, b, sched, 1e-9, 60)
    assert abs(res.n_iterations - rr.n_iterations) <= 1
    k = min(res.n_iterations, rr.n_iterations)
    assert res.orders[:k] == rr.orders[:k]
    assert rel_l2(res.x, rr.x) <= 1e-6


def test_gmres_with_an_arbitrary_callable_runs_the_reference_loop():
    from oracle import fmm_oracle as O
    from paper_1506_05957_b200.solver import RelaxationSchedule, gmres

    op, ref = _ops("laplace_second")
    b = ref.apply(np.ones(op.shape[0]), 12)
    seen = []
    res = gmres(lambda v, p: op.apply(v, p), b, RelaxationSchedule(10, 3, 1e-6, True), tol=1e-6,
                max_iter=50, callback=lambda k, r, p: seen.append(p))
    dev = gmres(op.apply, b, RelaxationSchedule(10, 3, 1e-6, True), tol=1e-6, max_iter=50)
    assert res.orders == dev.orders == seen
    assert rel_l2(res.x, dev.x) <= 1e-10
    rr = O.gmres(ref.apply, b, O.RelaxationSchedule(10, 3, 1e-6, True), 1e-6, 50)
    assert rel_l2(res.x, rr.x) <= 1e-6


def test_apply_device_is_ordered_on_the_callers_stream():
    import torch

    op, _ = _ops("laplace_second", level=3, n_crit=64)
    n = op.shape[0]
    x = np.random.default_rng(2).uniform(-1.0, 1.0, n)
    want = op.apply(x, 8)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        xd = torch.zeros(n, dtype=torch.float64, device="cuda")
        yd = torch.zeros(n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            # x is written on `s` right before the apply: a racing apply would read zeros
            xd.copy_(torch.from_numpy(x).cuda(non_blocking=False))
            xd.mul_(2.0)
            xd.mul_(0.5)
            op.apply_device(xd.data_ptr(), yd.data_ptr(), 8, stream=s.cuda_stream)
            yd.mul_(1.0)  # queued behind the apply on s
        s.synchronize()
    assert rel_l2(yd.cpu().numpy(), want) <= 1e-13
    # NULL stream: ordered after the legacy default stream, synchronous
    xd2 = torch.from_numpy(x).cuda()
    yd2 = torch.zeros_like(xd2)
    op.apply_device(xd2.data_ptr(), yd2.data_ptr(), 8)
    assert rel_l2(yd2.cpu().numpy(), want) <= 1e-13


def test_two_operators_on_the_same_device_and_graph_regrowth():
    # order tables regrow when a higher p follows lower ones; the cached lower-p graphs must
    # see the new layout (graph signature includes the table sizes)
    op, ref = _ops("laplace_second", level=3, n_crit=64)
    x = np.random.default_rng(9).uniform(-1.0, 1.0, op.shape[0])
    y4 = op.apply(x, 4)
    op.assemble_rhs(np.ones(op.shape[0]))  # p = 18 tables
    op.apply(x, 16)
    assert rel_l2(op.apply(x, 4), ref.apply(x, 4)) <= 1e-10
    assert rel_l2(op.apply(x, 4), y4) <= 1e-14
