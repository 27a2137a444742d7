"""GPU: the partitioned (multi-GPU) apply, checked on one GPU.

* virtual shards (no collectives): every rank's restricted work lists produce
  exactly its own rows of the unpartitioned mat-vec (bitwise, same kernels and
  summation order), for several world sizes;
* a real NCCL shard with world size 1 (all-gathers of the leaf multipoles and
  of y are then copies): full mat-vec and relaxed GMRES unchanged.
Kernels of different ranks never wait on each other here (see the profiling
recipe); the N>1 collectives are covered by construction plus the CPU gloo tests.
"""

import numpy as np
import pytest

from conftest import load_golden, rel_l2

pytestmark = pytest.mark.gpu


def _op(name):
    from paper_1506_05957_b200 import meshes as M
    from paper_1506_05957_b200.configs import CONFIGS
    from paper_1506_05957_b200.operator import GpuBemOperator

    cfg = CONFIGS[name]
    g = load_golden(name)
    mesh = M.Mesh(g["vertices"], g["triangles"]) if "vertices" in g else cfg.mesh()
    return GpuBemOperator(mesh, cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu), cfg, g


@pytest.mark.parametrize("name", ["cfg1", "stokes_ico3", "cfg2"])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_virtual_shards_reassemble_the_matvec(name, world):
    from paper_1506_05957_b200.parallel import leaf_bounds

    op, cfg, g = _op(name)
    x = g["x"]
    full = op.apply(x, cfg.p_initial)
    tb, sb = leaf_bounds(op, world)
    nc = 3 if cfg.formulation == "stokes" else 1
    y = np.full(op.shape[0], np.nan)
    for r in range(world):
        op.shard(r, world, tb, sb, None)
        part = op.apply(x, cfg.p_initial)
        rows = op.owned_panels(tb, r)
        idx = (rows[:, None] * nc + np.arange(nc)[None, :]).ravel()
        y[idx] = part[idx]
    op.unshard()
    assert not np.any(np.isnan(y))
    np.testing.assert_array_equal(y, full)
    assert rel_l2(op.apply(x, cfg.p_initial), full) == 0.0  # unshard restores the full apply


def test_nccl_world1_shard_matches_and_solves():
    from paper_1506_05957_b200.parallel import leaf_bounds, nccl_unique_id
    from paper_1506_05957_b200.solver import solve

    op, cfg, g = _op("cfg2")
    x = g["x"]
    ref = op.apply(x, 12)
    tb, sb = leaf_bounds(op, 1)
    op.shard(0, 1, tb, sb, nccl_unique_id())
    # the sharded upward pass is P2M + M2M (the unsharded one direct): equal to roundoff
    assert rel_l2(op.apply(x, 12), ref) <= 1e-13
    res = solve(op, g["rhs"], eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min)
    assert res.orders == g["relaxed_orders"].tolist()
    assert rel_l2(res.x, g["relaxed_x"]) <= 1e-6
    op.unshard()


def test_leaf_work_weights_are_positive_and_complete():
    op, _, _ = _op("cfg2")
    wt, ws = op.leaf_work("tgt"), op.leaf_work("src")
    assert len(wt) == op.plan.n_tgt_leaves and len(ws) == op.plan.n_src_leaves
    assert np.all(wt > 0) and np.all(ws > 0)
    assert ws.sum() == len(op.src_pos)


def test_virtual_shard_refuses_gmres():
    from paper_1506_05957_b200.parallel import leaf_bounds
    from paper_1506_05957_b200.solver import solve

    op, cfg, g = _op("cfg1")
    tb, sb = leaf_bounds(op, 2)
    op.shard(0, 2, tb, sb, None)
    with pytest.raises(ValueError, match="virtual shard"):
        solve(op, g["rhs"], eta=1e-6, p_initial=10, p_min=3)
    op.unshard()
