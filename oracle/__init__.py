"""CPU oracle for the relaxed-GMRES FMM-BEM hot path — TEST INFRASTRUCTURE ONLY.

``fmm_oracle`` restates, in numpy/scipy, the algorithm of the reference
package (``/root/reference/pkg/src/fmmbem``: octree.py, fmm.py, harmonics.py,
bemop.py, quadrature.py, solver.py), citing file:line per function.  It is the
checker for the CUDA path and the CPU baseline leg of ``bench.py``; only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import it.  The product
(``paper_1506_05957_b200``) never imports it.

Parity pin: the oracle is checked against golden vectors produced by running
the reference itself in the build container (``tools/make_goldens.py`` ->
``tests/golden/*.npz``; test: ``tests/test_oracle.py``): bitwise trees and
pair sets, correction matrices to 1e-12, mat-vecs at equal p to 1e-10, GMRES
histories.  The reference is pure Python, so there is no compiled
``oracle/_ref``; the reference cannot travel to the GPU box, the goldens do.
"""
