"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for parity checking.

This package is a float64 numpy restatement of the reference ``odegrad``
gradient path (``/root/reference/pkg/src/odegrad``), batched over independent
samples (rows).  It is imported only by ``tests/``, ``__graft_entry__.smoke()``
(as the checker) and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs.  The product path (``paper_2206_01298_b200``) never imports it and has
no CPU fallback.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by running the reference itself in the build
container (``tools/make_golden.py`` -> ``tests/golden/*.npz``) and against the
reference test-suite's known-answer values.  The C3 (conv) and C4 (CNF)
right-hand sides have no reference counterpart; their restatements are pinned
by finite differences and the adjoint identity only.
"""
