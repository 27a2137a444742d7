"""B200-native hot path of the relaxed-GMRES FMM-BEM solver (arXiv:1506.05957).

Drop-in for the reference's ``BemOperator.apply(x, p)`` / ``solve`` surface
(``pkg/src/fmmbem/bemop.py:272``, ``solver.py:137``); the mat-vec, the octree,
the traversal, the near/singular correction and the GMRES loop run as
hand-written sm_100a CUDA kernels in ``libfmmbem_b200.so`` behind a C ABI
(``include/fmmbem_b200.h``).
"""

from .meshes import Mesh, make_icosphere, make_octasphere, make_rbc, make_rbc_lattice, read_mesh, write_mesh

__all__ = ["Mesh", "make_icosphere", "make_octasphere", "make_rbc", "make_rbc_lattice",
           "read_mesh", "write_mesh"]
