"""CPU oracle for arXiv 2012.09646 (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under
``oracle/``.  The product path (``paper_2012_09646_b200``) never imports,
links or executes it, and this package imports nothing from the product --
the two share only the seeded input generator ``synth``.

Contents
* ``oracle.dag``   -- brute-force pairwise read/write-conflict DAG builder,
  stream-assignment and transfer oracles (§IV-A, §IV-C
  L559-664; readings D1-D8 in DESIGN.md).
* ``oracle.vec``, ``oracle.bs``, ``oracle.img``, ``oracle.ml``,
  ``oracle.hits``, ``oracle.dl`` -- serial fp64 implementations of the six
  benchmarks (§V-B), written as plain numpy in the paper's
  order; every function cites the passage it follows.

Pinning status is stated per module header and collected in DESIGN.md
"Oracle pins".  Constants the paper does not fix are marked "parity
unpinned (constant)" -- they are readings, pinned only for self-consistency.
"""
