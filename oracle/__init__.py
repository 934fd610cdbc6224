"""CPU oracle for the KaaS hot path -- TEST INFRASTRUCTURE ONLY.

A plain-Python/numpy restatement of the reference executor path
(arXiv 2212.08146 artifact, ``pkg/src/kaas``): the executor lifecycle and
buffer-cache ledger (``executor.py``), the builtin kernels and timing model
(``backend.py``), and the router policies (``router.py``), plus CPU
definitions of the two new library kernels (``cgemm``, ``jacobi_sweep``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the CPU arm -- never as the thing measured or shipped.  The product package
(``paper_2212_08146_b200``) never imports it.

Pinning: ``tests/golden/`` holds fixtures produced by running the real
reference (``tests/golden/make_golden.py``, run in the build container where
``/root/reference`` exists); ``tests/test_oracle.py`` checks this restatement
against them.  ``cgemm`` / ``jacobi_sweep`` have no reference implementation,
so their parity is pinned only by the north-star tolerances against float64
truth ("parity unpinned" at the reference level).
"""
