"""CPU: pin the oracle (oracle/fmm_oracle.py) and the host geometry against the
reference's own outputs (tests/golden, produced by tools/make_goldens.py)."""

import hashlib

import numpy as np
import pytest

from conftest import rel_l2

from oracle import fmm_oracle as O
from paper_1506_05957_b200 import meshes as M
from paper_1506_05957_b200.configs import CONFIGS
from paper_1506_05957_b200.geometry import PanelSet

SMALL = ["cfg1", "laplace1_ico3", "stokes_ico3", "rbc2"]


def _mesh(g, name):
    if "vertices" in g:
        return M.Mesh(g["vertices"], g["triangles"])
    return CONFIGS[name].mesh()


@pytest.mark.parametrize("name", ["cfg1", "laplace1_ico3", "stokes_ico3", "rbc2", "cfg2", "cfg3"])
def test_generators_reproduce_golden_meshes(golden, name):
    """The mesh generators are deterministic: regenerated meshes hash to the goldens'."""
    g = golden(name)
    mesh = CONFIGS[name].mesh()
    h = hashlib.sha256()
    h.update(mesh.vertices.tobytes())
    h.update(mesh.triangles.tobytes())
    assert h.hexdigest() == str(g["mesh_sha256"])
    assert M.is_closed(mesh) and mesh.volume > 0.0


@pytest.mark.parametrize("name", SMALL)
def test_host_geometry_is_bitwise_the_reference(golden, name):
    """Gauss points feed the exact-tie octree: they must equal the reference's bit for bit."""
    g = golden(name)
    ps = PanelSet(_mesh(g, name))
    assert np.array_equal(ps.src_pos, g["src_pos"])


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_host_geometry_hash_large(golden, name):
    g = golden(name)
    ps = PanelSet(_mesh(g, name))
    assert hashlib.sha256(ps.src_pos.tobytes()).hexdigest() == str(g["src_pos_sha256"])


_ORC = {}


def _oracle(golden, name):
    if name not in _ORC:
        cfg = CONFIGS[name]
        g = golden(name)
        _ORC[name] = O.OracleOperator(_mesh(g, name), cfg.formulation, theta=cfg.theta,
                                      n_crit=cfg.n_crit, mu=cfg.mu)
    return _ORC[name]


@pytest.mark.parametrize("name", ["cfg1", "stokes_ico3", "rbc2"])
def test_oracle_tree_and_pairs(golden, name):
    g = golden(name)
    op = _oracle(golden, name)
    for side, tree in (("src", op.plan.S), ("tgt", op.plan.T)):
        assert np.array_equal(tree.perm, g[side + "_perm"])
        key = lambda c, l: (int(l), *map(float, c))  # noqa: E731
        assert sorted(key(c, l) for c, l in zip(tree.center, tree.level)) == \
            sorted(key(c, l) for c, l in zip(g[side + "_center"], g[side + "_level"]))
    S, T = op.plan.S, op.plan.T
    for kind, pairs in (("m2l", op.plan.m2l_pairs), ("p2p", op.plan.p2p_pairs)):
        mine = {((int(S.level[s]), *S.center[s]), (int(T.level[t]), *T.center[t])) for s, t in pairs}
        ref = {((int(g["src_level"][s]), *g["src_center"][s]), (int(g["tgt_level"][t]), *g["tgt_center"][t]))
               for s, t in g[kind + "_pairs"]}
        assert mine == ref


@pytest.mark.parametrize("name", ["cfg1", "laplace1_ico3", "stokes_ico3"])
def test_oracle_correction_matches_reference(golden, name):
    import scipy.sparse as sp

    g = golden(name)
    op = _oracle(golden, name)
    B = sp.csr_matrix((g["csys_data"], g["csys_indices"], g["csys_indptr"]), shape=op.c_sys.shape)
    assert abs(op.c_sys - B).max() <= 1e-13 * abs(B).max()


@pytest.mark.parametrize("name,ps", [("cfg1", [1, 3, 6, 10, 12]), ("laplace1_ico3", [3, 10]),
                                     ("stokes_ico3", [5, 12]), ("rbc2", [5])])
def test_oracle_apply_matches_reference(golden, name, ps):
    g = golden(name)
    op = _oracle(golden, name)
    for p in ps:
        assert rel_l2(op.apply(g["x"], p), g[f"apply_p{p}"]) <= 1e-12


@pytest.mark.parametrize("name", ["cfg1", "laplace1_ico3"])
def test_oracle_dense_and_rhs(golden, name):
    g = golden(name)
    op = _oracle(golden, name)
    assert rel_l2(op.dense_apply(g["x"]), g["dense"]) <= 1e-13
    assert rel_l2(op.assemble_rhs(g["boundary_data"]), g["rhs"]) <= 1e-13


def test_oracle_gmres_history_matches_reference(golden):
    g = golden("cfg1")
    cfg = CONFIGS["cfg1"]
    op = _oracle(golden, "cfg1")
    r = O.gmres(op.apply, g["rhs"], O.RelaxationSchedule(cfg.p_initial, cfg.p_min, cfg.tol, True),
                cfg.tol, cfg.max_iter)
    assert r.orders == g["relaxed_orders"].tolist()
    np.testing.assert_allclose(r.residuals, g["relaxed_residuals"], rtol=1e-8)
    assert rel_l2(r.x, g["relaxed_x"]) <= 1e-12


def test_singular_laplace_known_answer():
    """Frozen self integral of 1/(4 pi r) over the reference test triangle
    (tests/test_quadrature.py:10-13,91-95 of the reference, rtol 1e-12)."""
    tri = np.array([[0.0, 0.0, 0.0], [1.1, 0.1, 0.0], [0.3, 0.9, 0.0]])
    assert np.isclose(O.singular_self("laplace_single", tri, 32), 0.19057608110821253, rtol=1e-12)


def test_stokeslet_self_block_is_rotation_covariant():
    tri = np.array([[0.0, 0.0, 0.0], [1.1, 0.1, 0.0], [0.3, 0.9, 0.0]])
    from scipy.spatial.transform import Rotation

    Q = Rotation.from_euler("xyz", [0.3, -1.1, 0.7]).as_matrix()
    a = O.singular_self("stokeslet", tri, 32)
    b = O.singular_self("stokeslet", tri @ Q.T, 32)
    np.testing.assert_allclose(b, Q @ a @ Q.T, atol=1e-13)


def test_harmonics_addition_theorem():
    """1/|x - y| = sum R_n^m(y) conj(I_n^m(x)) for |y| < |x| (harmonics.py:11)."""
    rng = np.random.default_rng(3)
    y = rng.uniform(-0.3, 0.3, (5, 3))
    x = rng.uniform(1.5, 2.0, (5, 3))
    p = 24
    R = O.solid_harmonics(y, p)
    Ir = O.solid_harmonics(x, p, irregular=True)
    approx = np.real(np.sum(R * np.conj(Ir), axis=1))
    np.testing.assert_allclose(approx, 1.0 / np.linalg.norm(x - y, axis=1), rtol=1e-12)


@pytest.mark.parametrize("name,ps", [("cfg1", [3, 10]), ("stokes_ico3", [5, 9])])
def test_parallel_oracle_equals_serial_oracle(name, ps):
    """oracle/parallel_oracle.py (the CPU timing legs) computes the oracle's apply item for item."""
    from oracle import fmm_oracle as O
    from oracle.parallel_oracle import ParallelOracle
    from paper_1506_05957_b200.configs import CONFIGS

    cfg = CONFIGS[name]
    op = O.OracleOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
    par = ParallelOracle(op, ps, workers=2)
    try:
        x = np.random.default_rng(1).uniform(-1.0, 1.0, op.n)
        for p in ps:
            y0, y1 = op.apply(x, p), par.apply(x, p)
            assert np.linalg.norm(y1 - y0) <= 1e-13 * np.linalg.norm(y0), p
    finally:
        par.close()


def test_expansion_goldens_are_consistent_with_the_oracle_harmonics():
    """tests/golden/expansion.npz (reference single-expansion API) vs the oracle's restated
    harmonics: P2M = q @ R, dipole P2M via the gradient shift rules, M2M via _mat_rconv."""
    from conftest import load_golden

    g = load_golden("expansion")
    src, q, nrm = g["src"], g["q"], g["nrm"]
    for p in (0, 3, 8, 14):
        R = O.solid_harmonics(src, p)
        assert np.allclose(q @ R, g[f"p2m_q_p{p}"], rtol=0, atol=1e-13)
        gx, gy, gz = O.regular_grad(R, p)
        d = q[:, None] * nrm
        assert np.allclose(d[:, 0] @ gx + d[:, 1] @ gy + d[:, 2] @ gz, g[f"p2m_d_p{p}"], atol=1e-13)
        T = O._mat_rconv(O.solid_harmonics(np.array([[-0.3, 0.2, -0.1]]), p)[0], p, "m2m")
        assert np.allclose(g[f"p2m_q_p{p}"] @ T.T, g[f"m2m_p{p}"], atol=1e-13)
