"""Mesh files written by the UNMODIFIED reference's write_mesh (mesh.py:175-184) for two of
this package's meshes (an icosphere and a rotated RBC pair with tags), for the ASCII
round-trip tests (tests/test_meshio.py).

Usage: PYTHONPATH=/root/reference/pkg/src:. python tools/make_golden_meshfile.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1506_05957_b200 import make_icosphere  # noqa: E402
from paper_1506_05957_b200.configs import _rbc_pair  # noqa: E402
from tools.make_goldens import OUT  # noqa: E402


def main():
    import fmmbem
    from fmmbem import mesh as RM

    ico = make_icosphere(2)
    RM.write_mesh(os.path.join(OUT, "ico2_ref.mesh"), fmmbem.Mesh(ico.vertices, ico.triangles))
    pair = _rbc_pair()
    tags = np.repeat(np.arange(2), pair.n_panels // 2)
    RM.write_mesh(os.path.join(OUT, "rbc2_ref.mesh"), fmmbem.Mesh(pair.vertices, pair.triangles, tags))
    back = RM.read_mesh(os.path.join(OUT, "rbc2_ref.mesh"))
    assert np.array_equal(back.tags, tags)
    print("wrote ico2_ref.mesh, rbc2_ref.mesh")


if __name__ == "__main__":
    main()
