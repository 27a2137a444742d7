"""Repeated applies (all orders) and solves, checking bitwise reproducibility: a soak test
for the persistent near-field kernel's stage hand-off.  python tools/stress_apply.py cfg2 500"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1506_05957_b200.configs import CONFIGS  # noqa: E402
from paper_1506_05957_b200.operator import GpuBemOperator  # noqa: E402

name, reps = sys.argv[1], int(sys.argv[2])
cfg = CONFIGS[name]
op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
x = np.random.default_rng(2).uniform(-1, 1, op.shape[0])
ref = {p: op.apply(x, p) for p in range(cfg.p_min, cfg.p_initial + 1)}
t0 = time.time()
bad = 0
for r in range(reps):
    p = cfg.p_min + r % (cfg.p_initial - cfg.p_min + 1)
    if not np.array_equal(op.apply(x, p), ref[p]):
        bad += 1
print(name, "applies", reps, "non-reproducible", bad, "seconds", round(time.time() - t0, 1))
sys.exit(1 if bad else 0)
