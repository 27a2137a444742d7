"""Generate golden fixtures by running the REFERENCE itself (this container only).

Usage:  PYTHONPATH=/root/reference/pkg/src:. python tools/make_goldens.py [case ...]

The reference (``/root/reference/pkg/src/fmmbem``, pure Python) is imported
unmodified and fed the exact mesh arrays this package generates; every array
it returns is written to ``tests/golden/<case>.npz``.  The GPU parity tests
and the CPU oracle tests compare against these files; ``/root/reference`` is
never read at test time (it does not exist on the GPU box).

Per case (see ``paper_1506_05957_b200.configs``):
  geometry      src_pos (bitwise check of the host geometry path)
  tree          perm / center / half_width / level / body_start / body_count / is_leaf
                for source and target trees (octree.py:57-131)
  traversal     m2l_pairs, p2p_pairs in reference cell numbering (fmm.py:84-125)
  correction    near pairs and the CSR of C_sys / C_rhs (bemop.py:95-184)
  apply         x = default_rng(1).uniform(-1, 1, n); apply(x, p) per p (bemop.py:272)
  dense         dense_apply(x) (bemop.py:276) for the small cases
  rhs           assemble_rhs(data) (bemop.py:290)
  solve         relaxed (and fixed) GMRES residuals / orders / x (solver.py:69-143)
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from paper_1506_05957_b200.configs import CONFIGS  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")

PLAN = {
    # name: (apply p list, dense?, tree+pairs?, correction?, fixed solve?, far/near parts?)
    "cfg1": dict(ps=list(range(1, 13)), dense=True, tree=True, corr=True, fixed=True, parts=True),
    "laplace1_ico3": dict(ps=[3, 6, 10], dense=True, tree=False, corr=True, fixed=False, parts=True),
    "stokes_ico3": dict(ps=[5, 8, 12], dense=True, tree=True, corr=True, fixed=False, parts=True),
    "rbc2": dict(ps=[5, 12], dense=False, tree=True, corr=False, fixed=False, parts=False),
    "cfg2": dict(ps=[3, 12], dense=False, tree=True, corr=False, fixed=True, parts=False),
    "cfg3": dict(ps=[5, 12], dense=False, tree=False, corr=False, fixed=False, parts=False),
}


def mesh_digest(mesh) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(mesh.vertices, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(mesh.triangles, dtype=np.int64).tobytes())
    return h.hexdigest()


def tree_arrays(prefix, tree, out):
    out[prefix + "perm"] = tree.perm.astype(np.int64)
    out[prefix + "center"] = tree.center
    out[prefix + "half"] = tree.half_width
    out[prefix + "level"] = tree.level.astype(np.int32)
    out[prefix + "body_start"] = tree.body_start.astype(np.int64)
    out[prefix + "body_count"] = tree.body_count.astype(np.int64)
    out[prefix + "is_leaf"] = tree.is_leaf


def make_case(name: str):
    import fmmbem
    from fmmbem.bemop import BemOperator

    cfg = CONFIGS[name]
    plan = PLAN[name]
    mesh = cfg.mesh()
    rmesh = fmmbem.Mesh(mesh.vertices, mesh.triangles)
    out = {}
    small = mesh.n_panels <= 2048
    out["mesh_sha256"] = np.array(mesh_digest(mesh))
    if small:
        out["vertices"] = mesh.vertices
        out["triangles"] = mesh.triangles
    t0 = time.perf_counter()
    op = BemOperator(rmesh, cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
    print(f"[{name}] setup {time.perf_counter() - t0:.1f}s", flush=True)
    if small:
        out["src_pos"] = op.src_pos
    else:
        h = hashlib.sha256(np.ascontiguousarray(op.src_pos).tobytes()).hexdigest()
        out["src_pos_sha256"] = np.array(h)
    if plan["tree"]:
        tree_arrays("src_", op.plan.src_tree, out)
        tree_arrays("tgt_", op.plan.tgt_tree, out)
        out["m2l_pairs"] = op.plan.m2l_pairs.astype(np.int64)
        out["p2p_pairs"] = op.plan.p2p_pairs.astype(np.int64)
        out["interaction_counts"] = op.plan.interaction_counts()
    if plan["corr"]:
        out["near_pairs"] = op._near_pairs.astype(np.int64)
        mats = [("csys", op._c_sys)]
        if cfg.formulation != "stokes":  # the stresslet C_rhs is 9x the size; RHS output pins it
            mats.append(("crhs", op._c_rhs))
        for key, mat in mats:
            m = mat.tocsr()
            m.sort_indices()
            out[key + "_indptr"] = m.indptr.astype(np.int64)
            out[key + "_indices"] = m.indices.astype(np.int64)
            out[key + "_data"] = m.data
    n = op.shape[0]
    x = np.random.default_rng(1).uniform(-1.0, 1.0, n)
    out["x"] = x
    for p in plan["ps"]:
        t0 = time.perf_counter()
        out[f"apply_p{p}"] = op.apply(x, p)
        print(f"[{name}] apply p={p} {time.perf_counter() - t0:.2f}s", flush=True)
    if plan["dense"]:
        out["dense"] = op.dense_apply(x)
    if plan["parts"]:
        _parts(op, x, plan["ps"][-1], out)
    data = cfg.boundary_data(op.centroids, op.normals)
    out["boundary_data"] = np.asarray(data)
    t0 = time.perf_counter()
    b = op.assemble_rhs(data)
    print(f"[{name}] rhs {time.perf_counter() - t0:.1f}s", flush=True)
    out["rhs"] = b
    for relaxed in ((True, False) if plan["fixed"] else (True,)):
        t0 = time.perf_counter()
        res = fmmbem.solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min,
                           relaxed=relaxed, max_iter=cfg.max_iter)
        tag = "relaxed" if relaxed else "fixed"
        print(f"[{name}] {tag} solve {time.perf_counter() - t0:.1f}s iters={res.n_iterations} "
              f"orders={res.orders}", flush=True)
        out[f"{tag}_residuals"] = np.asarray(res.residuals)
        out[f"{tag}_orders"] = np.asarray(res.orders, dtype=np.int64)
        out[f"{tag}_x"] = res.x
        out[f"{tag}_converged"] = np.array(res.converged)
        if cfg.formulation == "stokes":
            out[f"{tag}_drag"] = op.drag_force(res.x)
        ex = cfg.exact_potential(op.centroids)
        if ex is not None:
            out[f"{tag}_err_exact"] = np.array(np.linalg.norm(res.x - ex) / np.linalg.norm(ex))
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"[{name}] wrote {len(out)} arrays", flush=True)


def _parts(op, x, p, out):
    """far_field / near_field of the operator's own channel data (fmm.py:203-419)."""
    from fmmbem.fmm import _stokeslet_channels
    from fmmbem.bemop import Formulation

    out["parts_p"] = np.array(p)
    if op.formulation is Formulation.STOKES:
        t = x.reshape(op.n_panels, 3)
        strengths = op.src_weight[:, None] * t[op.src_panel]
        q = _stokeslet_channels(op.src_pos, strengths)
        pot, grad = op.plan.far_field(charges=q, p=p, want_gradient=True)
        npot, ngrad = op.plan.near_field(charges=q, want_gradient=True)
        out.update(far_pot=pot, far_grad=grad, near_pot=npot, near_grad=ngrad, channels_q=q)
        return
    charges = op.src_weight * x[op.src_panel]
    if op.formulation is Formulation.LAPLACE_SECOND:
        dip = charges[:, None] * op.src_normal
        out["far_pot"] = op.plan.far_field(dipoles=dip, p=p)
        out["near_pot"] = op.plan.near_field(dipoles=dip)
    else:
        out["far_pot"] = op.plan.far_field(charges=charges, p=p)
        out["near_pot"] = op.plan.near_field(charges=charges)


if __name__ == "__main__":
    names = sys.argv[1:] or list(PLAN)
    for nm in names:
        make_case(nm)
