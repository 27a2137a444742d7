"""One relaxed solve of a config (for an ncu launch list of the whole solve).

python tools/solve_launches.py cfg4
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1506_05957_b200.configs import CONFIGS  # noqa: E402
from paper_1506_05957_b200.operator import GpuBemOperator  # noqa: E402
from paper_1506_05957_b200.solver import solve  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
b = op.assemble_rhs(cfg.boundary_data(op.centroids, op.normals))
r = solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min, relaxed=True, max_iter=cfg.max_iter)
print(sys.argv[1], r.n_iterations, r.orders)
