"""Measurement helpers for bench.py and tools/ (host-side analysis only; no
method arithmetic, no device work):

* ``critical_path`` -- longest vertex-weighted path of an inferred DAG;
* ``dag_rooflines`` -- SURVEY §8(d) "Rooflines reported per DAG":
  R_cp = max over root->sink paths of the vertex bytes at HBM bandwidth
  (north_star's "slowest branch's bytes at HBM bandwidth"), R_work = all
  vertex bytes at HBM bandwidth (the stronger bound when branches contend);
* ``contention_free`` -- the paper's Fig. 9 estimate (§V-E
  L1195-1201): per-vertex times measured under SERIAL scheduling (each
  kernel alone on the GPU) summed along the DAG's longest path;
* ``overlap`` -- the paper's CT / TC / CC / TOT overlap metrics (§V-F
  L1265-1291) of an execution timeline.
"""
from __future__ import annotations


def critical_path(n, edges, weight):
    """Longest path (sum of vertex weights) over vertices 0..n-1 of a DAG
    whose edges (p, c, ...) all have p < c (ids are issue order)."""
    best = [0.0] * n
    preds = [[] for _ in range(n)]
    for e in edges:
        preds[e[1]].append(e[0])
    for v in range(n):
        best[v] = weight[v] + max((best[p] for p in preds[v]), default=0.0)
    return max(best, default=0.0)


def kernel_vertices(verts):
    """Ids of the kernel vertices of an exported DAG, in issue order."""
    return [v[0] for v in verts if v[1] == "kernel"]


def dag_rooflines(verts, edges, vertex_bytes, bw_gbs, vertex_floor_ms=None):
    """(R_cp ms, R_work ms) of one DAG.

    ``vertex_bytes``: algorithmic HBM bytes of each KERNEL vertex in issue
    order (the program's ``kernel_bytes()`` values).  ``vertex_floor_ms``
    (optional, same order): a non-HBM lower bound per kernel (B&S: FP64
    pipe time); a vertex then weighs max(bytes / bw, floor).  R_work is
    max(total bytes / bw, total floor) -- both resources are shared."""
    kv = kernel_vertices(verts)
    if len(kv) != len(vertex_bytes):
        raise ValueError(f"{len(kv)} kernel vertices vs {len(vertex_bytes)} byte counts")
    n = max((v[0] for v in verts), default=-1) + 1
    w = [0.0] * n
    for i, v in enumerate(kv):
        t = vertex_bytes[i] / (bw_gbs * 1e9) * 1e3
        if vertex_floor_ms is not None:
            t = max(t, vertex_floor_ms[i])
        w[v] = t
    r_cp = critical_path(n, edges, w)
    r_work = sum(vertex_bytes) / (bw_gbs * 1e9) * 1e3
    if vertex_floor_ms is not None:
        r_work = max(r_work, sum(vertex_floor_ms))
    return r_cp, r_work


def contention_free(verts, edges, kernel_ms, host_ms=None):
    """Fig. 9 contention-free time: the DAG's longest path with each kernel
    vertex weighted by its time under serial scheduling (plus the H2D copies
    it consumed, in stream mode) and each host vertex by its D2H time.
    ``kernel_ms``: per kernel vertex in issue order; ``host_ms``: {vertex id:
    ms} for host vertices."""
    kv = kernel_vertices(verts)
    n = max((v[0] for v in verts), default=-1) + 1
    w = [0.0] * n
    for i, v in enumerate(kv):
        w[v] = kernel_ms[i]
    for v, t in (host_ms or {}).items():
        w[v] = t
    return critical_path(n, edges, w)


def _union(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def _covered(a, b, u):
    s = 0.0
    for x, y in u:
        lo, hi = max(a, x), min(b, y)
        if hi > lo:
            s += hi - lo
    return s


def overlap(kernels, transfers):
    """Paper §V-F (L1272-1283) overlap metrics of a timeline; ``kernels`` and
    ``transfers`` are lists of (start, end).  CT = share of kernel time
    overlapping any transfer; TC = share of transfer time overlapping any
    kernel; CC = share of kernel time overlapping another kernel; TOT =
    share of all item time overlapping any other item (each overlapped
    instant counted once: unions of intervals)."""
    K, T = list(kernels), list(transfers)
    uT, uK = _union(T), _union(K)
    kt = sum(b - a for a, b in K)
    tt = sum(b - a for a, b in T)
    ct = sum(_covered(a, b, uT) for a, b in K) / kt if kt else 0.0
    tc = sum(_covered(a, b, uK) for a, b in T) / tt if tt else 0.0
    cc = sum(_covered(a, b, _union(K[:i] + K[i + 1:])) for i, (a, b) in enumerate(K)) / kt if kt else 0.0
    A = K + T
    tot = (sum(_covered(a, b, _union(A[:i] + A[i + 1:])) for i, (a, b) in enumerate(A)) / (kt + tt)
           if (kt + tt) else 0.0)
    span = (max(b for _, b in A) - min(a for a, _ in A)) if A else 0.0
    return {"CT": ct, "TC": tc, "CC": cc, "TOT": tot, "kernel_ms": kt, "transfer_ms": tt,
            "span_ms": span, "items": len(A)}
