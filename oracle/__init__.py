"""CPU oracle for the SlingBAG Pro forward/adjoint path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package, and only as the checker or the timed CPU baseline.  The product
package ``paper_2601_00551_b200`` never imports it and has no CPU fallback.

Modules
-------
radiator   FP64 numpy restatement of reference radiator.py:157-435 with the
           scratch-key collision fixed plus the detector
           directivity extension.
optimizer  restatement of reference optimizer.py (filter, Adam step, density
           control, hierarchical driver) on top of ``radiator``.
render     restatement of reference render.py:55-93 (voxelize) used for the
           volume-parity check.

Pinning: ``tests/golden/make_golden.py`` runs the reference itself (imported
from /root/reference with the cache-key rename applied) on seeded inputs and
freezes its outputs under ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks this oracle against every fixture.  Directivity modes other than
``none`` are not in the reference; they are pinned by (1) ``none`` equalling
the reference, (2) central finite differences, (3) the inner-product filter
identity.
"""
