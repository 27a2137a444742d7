"""Per-apply timeline of the concurrent step (FMMBEM_TIMELINE=1): when the basis stream, the M2M
levels, the M2L, the L2L and the near field end, relative to the apply's start (ms).

python tools/timeline.py [cfg] [p]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ["FMMBEM_TIMELINE"] = "1"
from paper_1506_05957_b200.configs import CONFIGS  # noqa: E402
from paper_1506_05957_b200.operator import GpuBemOperator  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
p = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.p_initial
op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, op.shape[0])).cuda()
y = torch.empty_like(x)
op.set_timing(True)
for _ in range(4):
    op.apply_device(x.data_ptr(), y.data_ptr(), p)
