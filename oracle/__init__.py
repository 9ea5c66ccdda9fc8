"""CPU oracle for the H-matrix assembly + H-matvec hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(``paper_1706_09384_b200``) imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import it, and there only as the checker /
the timed CPU baseline, never as the thing measured or shipped.

What it is
----------
A numpy restatement of the reference ``hmatx`` package
(``/root/reference/pkg/src/hmatx``) for the hot path:

* ``oracle.geometry``  -- cluster tree + block tree, restating
  ``geometry.py:94-295`` and the sphere generator ``geometry.py:310-344``.
  PINNED bit-exact against the reference module itself (tests import it when
  ``/root/reference`` is present) and against committed golden fixtures
  (``tests/golden/``, written by ``tests/golden/make_golden.py``).
* ``oracle.kernels``   -- Green's-tensor entries, restating
  ``_kernelcore_np.py:17-130`` with the same numpy operation order.
  PINNED bit-exact against the reference module and the golden fixtures.
* ``oracle.lowrank``   -- partially pivoted scalar ACA, sigma_3-pivoted vector
  ACA, randomized-SVD fallback and QR+SVD recompression.  The reference
  modules holding these (``lowrank.py``) are ABSENT from the mount; the code
  here restates SPEC.md:243-354 and PAPER.md:261-382,431-443 with the
  decisions of SURVEY.md 8(c) pinned.  Parity for this part is pinned only by
  the SPEC known-answer tests (rank-1 -> 1, zero -> 0, single 3x3 exact,
  idempotent recompression, <= 3 eps dense checks); there is no reference
  implementation or golden vector for it: "parity unpinned" beyond those KATs.
* ``oracle.hmatrix``   -- assemble / matvec / storage_report (
  reference ``hmatrix.py`` ABSENT -> pinned only by SPEC KATs).
* ``oracle.solve``     -- restarted GMRES (reference
  ``solve.py`` ABSENT -> pinned only by SPEC KATs and a scipy cross-check).
"""
