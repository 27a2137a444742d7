"""Where the end-to-end time of one relaxed solve goes (wall vs device events).

python tools/e2e_probe.py [cfg]"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1506_05957_b200 import _native as N
from paper_1506_05957_b200.configs import CONFIGS
from paper_1506_05957_b200.operator import GpuBemOperator
from paper_1506_05957_b200.solver import RelaxationSchedule, _device_gmres

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'cfg2']
op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
b = op.assemble_rhs(cfg.boundary_data(op.centroids, op.normals))
sched = RelaxationSchedule(p_initial=cfg.p_initial, p_min=cfg.p_min, eta=cfg.tol, relaxed=True)
bp = torch.from_numpy(np.ascontiguousarray(b)).pin_memory().numpy()
for _ in range(3):
    _device_gmres(op, bp, sched, cfg.tol, cfg.max_iter)
walls, calls = [], []
for _ in range(10):
    t = time.perf_counter()
    out = _device_gmres(op, bp, sched, cfg.tol, cfg.max_iter)
    walls.append(time.perf_counter() - t)
    calls.append(op.counters()[2])
print('host API: iters', out.n_iterations, 'wall ms', np.median(walls) * 1e3,
      'event ms (H2D..D2H)', np.median(calls))
lib = N.load()
bd = torch.from_numpy(b).cuda()
xd = torch.empty_like(bd)
res = np.zeros(cfg.max_iter)
ords = np.zeros(cfg.max_iter, dtype=np.int32)
nit, conv = ctypes.c_int32(0), ctypes.c_int32(0)
walls, calls = [], []
for _ in range(10):
    torch.cuda.synchronize()
    t = time.perf_counter()
    N.check(lib.fmmbem_op_gmres_device(op._h, ctypes.c_void_p(bd.data_ptr()), cfg.tol, cfg.tol, cfg.p_initial,
                                       cfg.p_min, 1, cfg.max_iter, ctypes.c_void_p(xd.data_ptr()),
                                       N.dptr(res), N.i32ptr(ords), ctypes.byref(nit), ctypes.byref(conv), None, None, None))
    walls.append(time.perf_counter() - t)
    calls.append(op.counters()[2])
print('device API: wall ms', np.median(walls) * 1e3, 'event ms', np.median(calls))
t = time.perf_counter()
for _ in range(10):
    x = np.empty(op.shape[0]); x[:] = bp
print('np.empty+copy ms', (time.perf_counter() - t) * 100)
t = time.perf_counter()
for _ in range(10):
    v = op._vec(bp)
print('_vec ms', (time.perf_counter() - t) * 100)
# the bench's e2e loop: L2 flush + sync before every timed call
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
walls, evs = [], []
for _ in range(10):
    flush.zero_()
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = _device_gmres(op, bp, sched, cfg.tol, cfg.max_iter)
    walls.append(time.perf_counter() - t)
    evs.append(op.counters()[2])
print('bench-style e2e: wall ms', np.median(walls) * 1e3, 'mean', np.mean(walls) * 1e3, 'event ms', np.median(evs))
t = time.perf_counter()
for _ in range(10):
    a = N.host_array(op.shape[0])
print('host_array ms', (time.perf_counter() - t) * 100)
