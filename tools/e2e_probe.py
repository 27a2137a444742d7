import time, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1506_05957_b200.configs import CONFIGS
from paper_1506_05957_b200.operator import GpuBemOperator
from paper_1506_05957_b200.solver import _device_gmres, RelaxationSchedule
cfg = CONFIGS['cfg2']
op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
b = op.assemble_rhs(cfg.boundary_data(op.centroids, op.normals))
sched = RelaxationSchedule(p_initial=12, p_min=3, eta=1e-6, relaxed=True)
bp = torch.from_numpy(np.ascontiguousarray(b)).pin_memory().numpy()
for _ in range(5): _device_gmres(op, bp, sched, 1e-6, 100)
walls, calls = [], []
for _ in range(30):
    t = time.perf_counter(); out = _device_gmres(op, bp, sched, 1e-6, 100); walls.append(time.perf_counter() - t)
    calls.append(op.counters()[2])
print('iters', out.n_iterations, 'wall us', np.median(walls)*1e6, 'event us (H2D..D2H)', np.median(calls)*1e3)
