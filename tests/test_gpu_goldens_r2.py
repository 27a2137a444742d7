"""GPU parity on the round-2 goldens from the unmodified reference (tools/make_goldens_r2.py).

* cfg2 apply at the relaxed solve's intermediate orders p = 5, 10 (full vectors).
* cfg5 apply at p = 10, 4 (the relaxed schedule's orders, sampled rows + norm).
* cfg4 apply at p = 8 and the relaxed GMRES solve of BASELINE config 4 (64 RBCs, 393 216
  unknowns, the only config where relaxation runs for many iterations): iteration count +-1,
  orders equal on the common prefix, solution <= 1e-6 on the sampled rows and in norm.
* both upward-pass modes (direct basis stream / leaf basis + M2M) give the same mat-vec.
Bars: BASELINE.json north_star (mat-vec <= 1e-10, iterations +-1, solution <= 1e-6).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel_l2

pytestmark = pytest.mark.gpu

_OPS = {}


def _op(name, upward=None, **env):
    """Operator of a config; upward / env select kernel variants (read at construction and at
    the first apply: FMMBEM_UPWARD direct|leaf, FMMBEM_DOWN path|l2l, FMMBEM_M2M grouped)."""
    from paper_1506_05957_b200.configs import CONFIGS
    from paper_1506_05957_b200.operator import GpuBemOperator

    key = (name, upward, tuple(sorted(env.items())))
    if key not in _OPS:
        cfg = CONFIGS[name]
        old = os.environ.pop("FMMBEM_UPWARD", None)
        if upward:
            os.environ["FMMBEM_UPWARD"] = upward
        try:
            _OPS[key] = (GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta,
                                        n_crit=cfg.n_crit, mu=cfg.mu), cfg)
        finally:
            os.environ.pop("FMMBEM_UPWARD", None)
            if old is not None:
                os.environ["FMMBEM_UPWARD"] = old
    return _OPS[key]


def _golden(name):
    if not os.path.exists(os.path.join(GOLDEN, f"{name}.npz")):
        pytest.skip(f"{name}.npz not generated")
    return load_golden(name)


@pytest.mark.parametrize("upward", ["direct", "leaf"])
def test_cfg2_intermediate_orders(upward):
    g = _golden("cfg2_mid")
    g0 = load_golden("cfg2")
    op, _ = _op("cfg2", upward)
    x = np.random.default_rng(1).uniform(-1.0, 1.0, op.shape[0])
    for p in (5, 10):
        assert rel_l2(op.apply(x, p), g[f"apply_p{p}"]) <= 1e-10, (upward, p)
    for p in (3, 12):
        assert rel_l2(op.apply(x, p), g0[f"apply_p{p}"]) <= 1e-10, (upward, p)


def test_upward_modes_agree_on_every_order():
    a, _ = _op("cfg2", "direct")
    b, _ = _op("cfg2", "leaf")
    x = np.random.default_rng(5).uniform(-1.0, 1.0, a.shape[0])
    for p in range(0, 15):
        assert rel_l2(b.apply(x, p), a.apply(x, p)) <= 1e-12, p


@pytest.mark.parametrize("upward", [None, "direct"])
def test_cfg5_intermediate_orders(upward):
    g = _golden("cfg5_mid")
    op, _ = _op("cfg5", upward)
    rows = g["rows"]
    x = np.random.default_rng(1).uniform(-1.0, 1.0, op.shape[0])
    for p in (10, 4):
        if f"apply_p{p}_rows" not in g:
            continue
        y = op.apply(x, p)
        assert rel_l2(y[rows], g[f"apply_p{p}_rows"]) <= 1e-10, p
        assert abs(np.linalg.norm(y) / float(g[f"apply_p{p}_norm"]) - 1.0) <= 1e-10, p


def test_cfg4_apply_p8():
    g = _golden("cfg4_solve")
    op, _ = _op("cfg4")
    rows = g["rows"]
    x = np.random.default_rng(1).uniform(-1.0, 1.0, op.shape[0])
    y = op.apply(x, 8)
    assert rel_l2(y[rows], g["apply_p8_rows"]) <= 1e-10
    assert abs(np.linalg.norm(y) / float(g["apply_p8_norm"]) - 1.0) <= 1e-10


def test_cfg4_relaxed_gmres_matches_reference():
    from paper_1506_05957_b200.solver import solve

    g = _golden("cfg4_solve")
    if "relaxed_orders" not in g:
        pytest.skip("cfg4 reference solve not finished")
    op, cfg = _op("cfg4")
    b = op.assemble_rhs(cfg.boundary_data(op.centroids, op.normals))
    assert abs(np.linalg.norm(b) / float(g["rhs_norm"]) - 1.0) <= 1e-10
    res = solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min, relaxed=True,
                max_iter=cfg.max_iter)
    ref_orders = [int(v) for v in g["relaxed_orders"]]
    assert res.converged == bool(g["relaxed_converged"])
    assert abs(res.n_iterations - len(ref_orders)) <= 1, (res.n_iterations, len(ref_orders))
    k = min(res.n_iterations, len(ref_orders))
    assert res.orders[:k] == ref_orders[:k]
    np.testing.assert_allclose(res.residuals[:k], g["relaxed_residuals"][:k], rtol=1e-5)
    assert rel_l2(res.x[g["rows"]], g["relaxed_x_rows"]) <= 1e-6
    assert abs(np.linalg.norm(res.x) / float(g["relaxed_x_norm"]) - 1.0) <= 1e-6
    drag = op.drag_force(res.x)
    assert np.linalg.norm(drag - g["drag"]) <= 1e-6 * np.linalg.norm(g["drag"])


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_downward_modes_agree(name):
    """Rotation L2L + leaf-only epilogue vs the path epilogue (L2L is exact): run in a
    subprocess each, since the mode switch is read once per process."""
    import subprocess
    import sys

    code = ("import numpy as np, sys; sys.path.insert(0, '.');"
            "from paper_1506_05957_b200.configs import CONFIGS;"
            "from paper_1506_05957_b200.operator import GpuBemOperator;"
            f"cfg = CONFIGS['{name}'];"
            "op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu);"
            "x = np.random.default_rng(1).uniform(-1, 1, op.shape[0]);"
            "np.save(sys.argv[1], np.stack([op.apply(x, p) for p in (3, 5, 12)]))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("path", "l2l"):
        f = os.path.join(root, "gpurun_out", f"down_{name}_{mode}.npy")
        os.makedirs(os.path.dirname(f), exist_ok=True)
        subprocess.run([sys.executable, "-c", code, f], cwd=root, check=True,
                       env=dict(os.environ, FMMBEM_DOWN=mode))
        out[mode] = np.load(f)
    for k in range(3):
        assert rel_l2(out["l2l"][k], out["path"][k]) <= 1e-12, k


@pytest.mark.parametrize("name,variant", [("cfg2", "1"), ("cfg3", "1"), ("cfg2", "1a")])
def test_shared_table_m2l_matches_reference_and_default(name, variant):
    """The shared-table rotation M2L (FMMBEM_M2L_SHARED=1: tables staged per CTA by bulk async
    copies, stage C on the transposed stage-A tables; 1a: the multipoles prefetched by cp.async)
    against the reference goldens and the default per-warp kernel, p = 3 .. 20 (every
    warps-per-CTA choice), 1 and 4 channels."""
    g = load_golden(name)
    op, _ = _op(name)
    x = np.random.default_rng(1).uniform(-1.0, 1.0, op.shape[0])
    base = {p: op.apply(x, p) for p in range(3, 21)}
    os.environ["FMMBEM_M2L_SHARED"] = variant
    try:
        from paper_1506_05957_b200.configs import CONFIGS
        from paper_1506_05957_b200.operator import GpuBemOperator

        cfg = CONFIGS[name]
        op2 = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
        for p in range(3, 21):
            y = op2.apply(x, p)
            assert rel_l2(y, base[p]) <= 1e-12, p
            if f"apply_p{p}" in g:
                assert rel_l2(y, g[f"apply_p{p}"]) <= 1e-10, p
    finally:
        os.environ.pop("FMMBEM_M2L_SHARED", None)


def test_basis_stream_kernels_agree():
    """The upward basis stream by bulk async copies (TMA ring, the default from 1 024 items) and by
    per-thread loads (FMMBEM_P2M=ldg) give the same mat-vec; the switch is read once per process,
    so each runs in a subprocess (cfg2: direct-basis mode, 85 k entries)."""
    import subprocess
    import sys

    code = ("import numpy as np, sys; sys.path.insert(0, '.');"
            "from paper_1506_05957_b200.configs import CONFIGS;"
            "from paper_1506_05957_b200.operator import GpuBemOperator;"
            "cfg = CONFIGS['cfg2'];"
            "op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu);"
            "x = np.random.default_rng(1).uniform(-1, 1, op.shape[0]);"
            "np.save(sys.argv[1], np.stack([op.apply(x, p) for p in (3, 5, 12, 16)]))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("tma", "ldg"):
        f = os.path.join(root, "gpurun_out", f"basis_{mode}.npy")
        os.makedirs(os.path.dirname(f), exist_ok=True)
        subprocess.run([sys.executable, "-c", code, f], cwd=root, check=True,
                       env=dict(os.environ, FMMBEM_P2M=mode))
        out[mode] = np.load(f)
    g = load_golden("cfg2")
    for i, p in enumerate((3, 5, 12, 16)):
        assert rel_l2(out["tma"][i], out["ldg"][i]) <= 1e-12, p
        if f"apply_p{p}" in g:
            assert rel_l2(out["tma"][i], g[f"apply_p{p}"]) <= 1e-10, p
