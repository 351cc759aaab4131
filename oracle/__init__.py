"""CPU oracle for the heightmap hot path -- TEST INFRASTRUCTURE ONLY.

This package restates the reference algorithm (``/root/reference/pkg``,
the pure-Python ``terrascout`` package) in plain numpy/scipy so parity can
be checked on the GPU box, where the reference tree does not exist.  Each
function cites the reference ``file:line`` it follows.

Who may use it: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` -- only as the
checker or the timed CPU baseline, never as the product path.  The product
package ``paper_2509_20198_b200`` never imports this package.

Pinning: ``tests/golden/make_golden.py`` imports the real reference in the
build container and writes seeded input/output vectors to
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this oracle
against every one of them (chunk points, positions/colours, Algorithm 1
rasters incl. face maps, conv/refine outputs, bake outputs, wire records).

Third-party arithmetic the reference delegates to (not under
/root/reference): scipy.spatial.Delaunay (Qhull) and cKDTree, numpy/OpenBLAS
sgemm, numpy.bincount.  Pinned de-facto versions: numpy 2.3.5, scipy
1.18.1 (this image).  The oracle calls Qhull exactly as the reference does
(``patches.py:319``); the NN rule is restated as the exact d^2 argmin with
lowest-index ties that the reference's own tests use
(``pkg/tests/test_patches.py:15-18``).
"""
