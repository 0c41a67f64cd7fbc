"""HITS oracle, serial fp64 (TEST INFRASTRUCTURE ONLY).

PAPER.md §V-B: "it computes the HITS algorithm on a graph [30]
(Kleinberg, L1604-1605) using repeated Sparse matrix-vector multiplication
(SpMV) on a matrix and its transpose".  Fig. 6 (L729-734) draws per
iteration SPMV x2, SUM x2, DIV x2, "[REPEAT...]".  Readings (DESIGN.md
R-HITS): A is the 0/1 adjacency matrix in CSR (values implicit 1), A^T a
second CSR; simultaneous update; the SUM node is the L2 norm (north_star:
"hub and authority vectors L2-normalised"); a1 = h1 = 1/sqrt(N) initially.

    a2 = A^T h1;  h2 = A a1;  an = ||a2||_2;  hn = ||h2||_2;  a1 = a2/an;  h1 = h2/hn

Pins (tests/test_oracle_hits.py): SpMV equals scipy.sparse products; norms
are 1 after each iteration; on small graphs with a spectral gap a and h
converge to the principal eigenvectors of A^T A and A A^T
(numpy.linalg.eigh); directed cycle -> uniform vectors; complete bipartite
K_{m,n} -> uniform authority on the sinks.
"""
import numpy as np

ITERATIONS = 10  # reading; parity unpinned (constant)


def spmv(row_ptr, col_idx, x):
    """y[i] = sum_{k in row i} x[col_idx[k]] (0/1 CSR, one row at a time)."""
    x = np.asarray(x, dtype=np.float64)
    n = len(row_ptr) - 1
    contrib = x[np.asarray(col_idx, dtype=np.int64)]
    rows = np.repeat(np.arange(n), np.diff(np.asarray(row_ptr, dtype=np.int64)))
    return np.bincount(rows, weights=contrib, minlength=n)


def l2norm(v):
    """SUM node read as the L2 norm: sqrt(sum v^2)."""
    v = np.asarray(v, dtype=np.float64)
    return float(np.sqrt(np.sum(v * v)))


def divide(v, nv):
    """DIV node: v / ||v||; a zero norm (empty graph) leaves zeros."""
    v = np.asarray(v, dtype=np.float64)
    return v / nv if nv > 0 else np.zeros_like(v)


def hits(row_ptr, col_idx, row_ptr_t, col_idx_t, iterations=ITERATIONS):
    n = len(row_ptr) - 1
    a1 = np.full(n, 1.0 / np.sqrt(n))
    h1 = np.full(n, 1.0 / np.sqrt(n))
    hist = []
    for _ in range(iterations):
        a2 = spmv(row_ptr_t, col_idx_t, h1)   # A^T h1
        h2 = spmv(row_ptr, col_idx, a1)       # A a1
        an = l2norm(a2)
        hn = l2norm(h2)
        a1 = divide(a2, an)
        h1 = divide(h2, hn)
        hist.append((an, hn))
    return dict(a1=a1, h1=h1, norms=hist, a2=a2, h2=h2)
