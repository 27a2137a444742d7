import sys, time, gc
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1506_05957_b200.configs import CONFIGS
from paper_1506_05957_b200.operator import GpuBemOperator
from paper_1506_05957_b200.solver import RelaxationSchedule, _device_gmres
cfg = CONFIGS['cfg5']
op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
b = op.assemble_rhs(cfg.boundary_data(op.centroids, op.normals))
sched = RelaxationSchedule(p_initial=cfg.p_initial, p_min=cfg.p_min, eta=cfg.tol, relaxed=True)
bp = torch.from_numpy(np.ascontiguousarray(b)).pin_memory().numpy()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
def loop(tag, keep, nogc, n=8):
    for _ in range(3): _device_gmres(op, bp, sched, cfg.tol, cfg.max_iter)
    if nogc: gc.disable()
    ms, held = [], []
    for _ in range(n):
        flush.zero_(); torch.cuda.synchronize()
        t = time.perf_counter()
        out = _device_gmres(op, bp, sched, cfg.tol, cfg.max_iter)
        t2 = time.perf_counter()
        ms.append(round(1e3*(t2-t),3))
        if keep: held.append(out)
    gc.enable()
    print(tag, ms)
for rep in range(2):
    loop('plain', False, False)
    loop('keep ', True, False)
    loop('nogc ', False, True)
# timing the free separately
for _ in range(3):
    out = _device_gmres(op, bp, sched, cfg.tol, cfg.max_iter)
    t = time.perf_counter(); out = None; print('free ms', 1e3*(time.perf_counter()-t))
