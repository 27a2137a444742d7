"""Build one config's operator and run a few mat-vecs (for ncu launch lists).

python tools/apply_once.py cfg5 14 [repeats]
"""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1506_05957_b200.configs import CONFIGS  # noqa: E402
from paper_1506_05957_b200.operator import GpuBemOperator  # noqa: E402

name, p = sys.argv[1], int(sys.argv[2])
rep = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = CONFIGS[name]
op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
x = np.random.default_rng(1).uniform(-1, 1, op.shape[0])
for _ in range(rep):
    y = op.apply(x, p)
print(name, p, float(np.linalg.norm(y)))
