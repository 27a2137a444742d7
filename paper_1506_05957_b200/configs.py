"""The five BASELINE.json configurations plus small parity cases.

Decisions for the spots where BASELINE.json and the reference disagree are
recorded in SURVEY.md Appendix C and DESIGN.md: icosphere meshes, the
reference's 19-point near rule and 32-node polar singular rule, unrestarted
GMRES (restart is moot at 2-4 iterations; config 4 raises max_iter),
n_crit = 128 where unstated, p_min = 3 (Laplace) / 5 (Stokes), Neumann data
q = -dphi/dn for the exterior second-kind Laplace problem
(``bemop.py:35-37,305-307``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import meshes as M

FOUR_PI = 4.0 * np.pi


def interior_charges(n: int, seed: int = 0, radius: float = 0.5) -> np.ndarray:
    """n points uniform in the ball |x| <= radius (seeded)."""
    rng = np.random.default_rng(seed)
    out = np.empty((n, 3))
    for i in range(n):
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        out[i] = v * radius * rng.uniform() ** (1.0 / 3.0)
    return out


def charge_potential(x: np.ndarray, charges: np.ndarray) -> np.ndarray:
    """phi(x) = sum_k 1 / (4 pi |x - x_k|)."""
    r = x[:, None, :] - charges[None, :, :]
    return np.sum(1.0 / (FOUR_PI * np.linalg.norm(r, axis=-1)), axis=1)


def charge_neumann(x: np.ndarray, normals: np.ndarray, charges: np.ndarray) -> np.ndarray:
    """q = -dphi/dn = sum_k (x - x_k).n / (4 pi r^3) (outward normal, exterior problem)."""
    r = x[:, None, :] - charges[None, :, :]
    d = np.linalg.norm(r, axis=-1)
    return np.sum(np.einsum("tki,ti->tk", r, normals) / (FOUR_PI * d ** 3), axis=1)


@dataclass
class Config:
    name: str
    mesh_fn: object
    formulation: str
    n_crit: int
    p_initial: int
    p_min: int
    tol: float
    theta: float = 0.5
    mu: float = 1e-3
    n_charges: int = 0
    seed: int = 0
    max_iter: int = 100
    extra: dict = field(default_factory=dict)

    def mesh(self):
        return self.mesh_fn()

    def boundary_data(self, centroids: np.ndarray, normals: np.ndarray):
        """Boundary data per the config (charges -> Neumann q; Stokes -> velocity)."""
        if self.formulation == "laplace_second":
            ch = interior_charges(self.n_charges, self.seed)
            return charge_neumann(centroids, normals, ch)
        if self.formulation == "laplace_first":
            ch = interior_charges(self.n_charges, self.seed)
            return charge_potential(centroids, ch)
        flow = self.extra.get("flow", "uniform")
        if flow == "shear":
            u = np.zeros((len(centroids), 3))
            u[:, 0] = centroids[:, 2]
            return u
        return np.tile([1.0, 0.0, 0.0], (len(centroids), 1))

    def exact_potential(self, centroids: np.ndarray):
        if self.formulation != "laplace_second":
            return None
        return charge_potential(centroids, interior_charges(self.n_charges, self.seed))


CONFIGS = {
    "cfg1": Config("cfg1", lambda: M.make_icosphere(3), "laplace_second", 64, 10, 3, 1e-6,
                   n_charges=1),
    "cfg2": Config("cfg2", lambda: M.make_icosphere(5), "laplace_second", 128, 12, 3, 1e-6,
                   n_charges=3),
    "cfg3": Config("cfg3", lambda: M.make_icosphere(5), "stokes", 128, 12, 5, 1e-5),
    "cfg4": Config("cfg4", lambda: M.make_rbc_lattice(4, 4, 1.0, 0), "stokes", 128, 12, 5, 1e-5,
                   max_iter=600, extra={"flow": "shear"}),
    "cfg5": Config("cfg5", lambda: M.make_icosphere(7), "laplace_second", 256, 14, 3, 1e-6,
                   n_charges=8),
    # small parity cases (committed goldens)
    "stokes_ico3": Config("stokes_ico3", lambda: M.make_icosphere(3), "stokes", 64, 12, 5, 1e-5),
    "laplace1_ico3": Config("laplace1_ico3", lambda: M.make_icosphere(3), "laplace_first", 64,
                            10, 3, 1e-6, n_charges=1),
    "rbc2": Config("rbc2", lambda: _rbc_pair(),
                   "stokes", 64, 12, 5, 1e-5, max_iter=200, extra={"flow": "shear"}),
}


def _rbc_pair():
    """Two level-3 cells (512 panels each) side by side: an iteration-heavy Stokes case."""
    from scipy.spatial.transform import Rotation

    rng = np.random.default_rng(0)
    cell = M.make_rbc(3)
    pitch = 2.0 * M.RBC_SCALE + 1.0
    verts, tris, off = [], [], 0
    for i in range(2):
        v = Rotation.random(rng=rng).apply(cell.vertices) + np.array([pitch * i, 0.0, 0.0])
        verts.append(v)
        tris.append(cell.triangles + off)
        off += len(v)
    return M.Mesh(np.vstack(verts), np.vstack(tris))
