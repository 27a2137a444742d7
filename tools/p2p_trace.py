"""Per-item clock trace of the persistent double-layer P2P kernel (FMMBEM_P2P_TRACE=1).

python tools/p2p_trace.py cfg2 12
Per CTA and item (globaltimer ns): producer (wait EMPTY, stage) and consumer (wait FULL, loop warp 0 / last warp,
reduce) phases in cycles; summarised over CTAs.
"""
import ctypes
import os
import sys

import numpy as np

os.environ.setdefault("FMMBEM_P2P_TRACE", "1")  # = stride: every stride-th item of a CTA is traced (32 slots)
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1506_05957_b200 import _native  # noqa: E402
from paper_1506_05957_b200.configs import CONFIGS  # noqa: E402
from paper_1506_05957_b200.operator import GpuBemOperator  # noqa: E402

name, p = sys.argv[1], int(sys.argv[2])
cfg = CONFIGS[name]
op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
x = np.random.default_rng(1).uniform(-1, 1, op.shape[0])
for _ in range(3):
    op.apply(x, p)
lib = _native.load()
buf = np.zeros(1024 * 32 * 8, dtype=np.int64)
lib.fmmbem_debug_p2p_trace.restype = ctypes.c_int
lib.fmmbem_debug_p2p_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.size))
t = buf.reshape(1024, 32, 8)
ctas = [c for c in range(1024) if t[c, 0, 3] != 0]
tot = {k: 0 for k in ("p_wait", "p_stage", "c_starve0", "c_starve", "c_busy", "span", "items")}
for c in ctas:
    items = [k for k in range(32) if t[c, k, 0] != 0 and t[c, k, 2] != 0]
    if not items:
        continue
    start = t[c, 0, 0]
    ends = [t[c, k, 7] for k in items]
    tot["span"] += max(ends) - start
    tot["items"] += len(items)
    prev_end = start
    for k in items:
        tot["p_wait"] += t[c, k, 1] - t[c, k, 0]
        tot["p_stage"] += t[c, k, 2] - t[c, k, 1]
        starve = max(0, t[c, k, 2] - prev_end)  # consumers idle until the producer staged item k
        tot["c_starve0" if k == 0 else "c_starve"] += starve
        tot["c_busy"] += t[c, k, 7] - max(prev_end, t[c, k, 2])
        prev_end = t[c, k, 7]
n = max(len(ctas), 1)
print(name, p, "ctas", len(ctas), {k: round(v / n) for k, v in tot.items()})
# globaltimer (ns): kernel-wide view
starts = np.array([t[c, 0, 0] for c in ctas])
ends = np.array([max(t[c, k, 7] for k in range(32) if t[c, k, 7] != 0) for c in ctas])
first_full = np.array([t[c, 0, 2] for c in ctas])
t0 = starts.min()
print("ns: cta start spread", int(starts.max() - t0), "first item staged (median)", int(np.median(first_full - t0)),
      "cta end min/median/max", int(ends.min() - t0), int(np.median(ends - t0)), int(ends.max() - t0))
last = sorted(((c, [int(t[c, k, 2] - t[c, k, 1]) for k in range(32) if t[c, k, 2]]) for c in ctas[:1]))
print("producer stage cycles per item (cta 0):", last)

# per traced item (mean over CTAs): producer wait / stage, consumer wait FULL / busy, ns
rows = []
for k in range(32):
    v = [(t[c, k, 1] - t[c, k, 0], t[c, k, 2] - t[c, k, 1], t[c, k, 4] - t[c, k, 3], t[c, k, 7] - t[c, k, 4])
         for c in ctas if t[c, k, 2] != 0 and t[c, k, 7] != 0 and t[c, k, 0] != 0]
    if v:
        rows.append((k, len(v)) + tuple(int(np.mean([r[j] for r in v])) for j in range(4)))
print("slot ctas p_wait p_stage c_waitfull c_busy (ns)")
for r in rows:
    print(*r)
