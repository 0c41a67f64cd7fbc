"""Brute-force DAG oracle (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Re-derives, by literally scanning every earlier op of a host-call trace, the
computation DAG the paper's scheduler infers at run time:

* PAPER.md §IV-A L386-430 and L490-491 (dependency sets, Fig. 3 A/B/C),
* L505-530 (host accesses as computational elements, Fig. 4 D),
* L546-558 (events, active computations, host-sync frontier),
* L570-582 + L647-654 (stream manager: FIFO reuse, first child on the
  parent's stream),

under the readings D1-D8 listed in DESIGN.md ("Readings of the paper").
It deliberately does NOT use the incremental last-writer/readers table of
the C++ scheduler: each dependency is found by an O(n^2 * args) scan.

Trace format (list of tuples):
  ("launch", name, [(array, mode), ...])   mode in {"R", "RW", "O"}
      "R"  = const/in pointer  (read-only, prefetched)
      "RW" = unannotated/inout pointer (modified, prefetched)
      "O"  = out pointer (modified, overwritten entirely: not prefetched)
  ("host", array, "R" | "W", off, nbytes)  host read / write of a byte range
  ("sync",)                                full barrier (build-only API, D6b)

Pinned by: tests/golden/*.dag (Appendix-A DAGs hand-derived from the
paper's figures), exhaustive tiny traces against the conflict-closure
invariant (tests/test_dag_oracle.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field


def merged_access(op):
    """Per-array dependency mode of one op: "W" if any use modifies it (D3)."""
    if op[0] == "launch":
        acc = {}
        for arr, mode in op[2]:
            m = "R" if mode == "R" else "W"
            if acc.get(arr) == "W":
                continue
            acc[arr] = m
        return acc
    if op[0] == "host":
        return {op[1]: op[2]}
    return {}


@dataclass
class DagResult:
    # recorded vertices: (vid, op_index, kind, name, stream)
    vertices: list = field(default_factory=list)
    # edges: set of (parent_vid, child_vid, array)
    edges: set = field(default_factory=set)
    # conflicts between recorded vertices (i<j share X, one writes, both active at j)
    conflicts: set = field(default_factory=set)
    # cross-stream waits: list of (child_vid, parent_vid)
    waits: list = field(default_factory=list)
    # host syncs: list of (host_vid or None, [parent vids waited on])
    host_waits: list = field(default_factory=list)


def build_dag(trace, stream_policy="fifo"):
    """Literal pairwise scan of the trace (SURVEY §8(c1) algorithm).

    ``stream_policy``: "fifo" = the paper's general policy (first child on
    the parent's stream, later children on other streams, L647-650);
    "single" = the paper's "simpler" policy, all children of a vertex on a
    single stream (L650-654): a vertex with parents goes on its lowest-id
    parent's stream.  The DAG (edges) does not depend on it."""
    accs = [merged_access(op) for op in trace]
    res = DagResult()
    vid_of = {}            # op index -> vertex id (recorded ops only)
    active = {}            # op index -> bool
    parents = {}           # op index -> set of op indices

    # stream oracle state
    stream_of = {}         # op index -> stream id
    tail = []              # stream -> last enqueued op index
    nactive = []           # stream -> number of active vertices

    def retire(op_idx):
        stack = [op_idx]
        while stack:
            k = stack.pop()
            if active.get(k):
                active[k] = False
                s = stream_of.get(k)
                if s is not None:
                    nactive[s] -= 1
            for p in parents.get(k, ()):
                if active.get(p):
                    stack.append(p)

    for j, op in enumerate(trace):
        if op[0] == "sync":
            for k in list(active):
                if active[k]:
                    retire(k)
            continue
        acc = accs[j]
        labels = {}  # parent op index -> set(arrays)
        for x, m in acc.items():
            # w* = last writer of x, active or not, host writes included
            wstar = None
            for k in range(j - 1, -1, -1):
                if accs[k].get(x) == "W":
                    wstar = k
                    break
            start = 0 if wstar is None else wstar + 1
            rd = [k for k in range(start, j)
                  if accs[k].get(x) == "R" and active.get(k, False)]
            if m == "R":
                if wstar is not None and active.get(wstar, False):
                    labels.setdefault(wstar, set()).add(x)
            else:
                if rd:
                    for k in rd:
                        labels.setdefault(k, set()).add(x)
                elif wstar is not None and active.get(wstar, False):
                    labels.setdefault(wstar, set()).add(x)

        if op[0] == "launch":
            vid = len(res.vertices)
            vid_of[j] = vid
            active[j] = True
            parents[j] = set(labels)
            # conflicts with every active recorded vertex (for the closure check)
            for k in range(j):
                if k in vid_of and active.get(k, False) and k != j:
                    if any(x in accs[k] and (accs[k][x] == "W" or m == "W")
                           for x, m in acc.items()):
                        res.conflicts.add((vid_of[k], vid))
            # stream oracle (SURVEY §8(c1) "Stream oracle")
            ps = sorted(labels, key=lambda k: vid_of[k])
            s = None
            if stream_policy == "single" and ps:
                s = stream_of[ps[0]]
            for p in ([] if s is not None else ps):
                sp = stream_of.get(p)
                if sp is not None and tail[sp] == p:
                    s = sp
                    break
            if s is None:
                for cand in range(len(tail)):
                    if nactive[cand] == 0:
                        s = cand
                        break
            if s is None:
                s = len(tail)
                tail.append(None)
                nactive.append(0)
            stream_of[j] = s
            tail[s] = j
            nactive[s] += 1
            res.vertices.append((vid, j, "kernel", op[1], s))
            for p in ps:
                for x in labels[p]:
                    res.edges.add((vid_of[p], vid, x))
                if stream_of[p] != s:
                    res.waits.append((vid, vid_of[p]))
        else:  # host access
            if labels:
                vid = len(res.vertices)
                vid_of[j] = vid
                parents[j] = set(labels)
                ps = sorted(labels, key=lambda k: vid_of[k])
                for k in range(j):
                    if k in vid_of and active.get(k, False):
                        x = op[1]
                        if x in accs[k] and (accs[k][x] == "W" or op[2] == "W"):
                            res.conflicts.add((vid_of[k], vid))
                res.vertices.append((vid, j, "host", op[1], -1))
                for p in ps:
                    for x in labels[p]:
                        res.edges.add((vid_of[p], vid, x))
                res.host_waits.append((vid, [vid_of[p] for p in ps]))
                for p in ps:
                    retire(p)
                active[j] = False  # synchronous CPU computation: done on return
            else:
                res.host_waits.append((None, []))
    return res


def closure(n, pairs):
    """Transitive closure of a relation on 0..n-1 given as (a, b) pairs, a<b."""
    succ = [set() for _ in range(n)]
    for a, b in pairs:
        succ[a].add(b)
    reach = [set() for _ in range(n)]
    for a in range(n - 1, -1, -1):
        for b in succ[a]:
            reach[a].add(b)
            reach[a] |= reach[b]
    return {(a, b) for a in range(n) for b in reach[a]}


def edge_pairs(res: DagResult):
    return {(p, c) for p, c, _ in res.edges}


def transfers(trace, has_host=None, nbytes=None):
    """Transfer oracle (SURVEY §8(c) "Transfer oracle").

    Arrays start device-valid (state "D" = device is the newest copy, host
    mirror stale) unless listed otherwise by the caller via host writes.
    Returns the ordered list of copies:
      ("H2D", array, bytes, launch_op_index)  before the first GPU use that
                                             reads an array whose newest copy
                                             is on the host;
      ("D2H", array, bytes, host_op_index)   for every host read while the
                                             device copy is newer (range bytes);
                                             a partial host write of a
                                             device-newer array first pulls
                                             the whole array.
    ``has_host[a]`` False means the array has no host mirror: host accesses
    then copy the range directly (H2D for writes, D2H for reads).
    ``nbytes[a]`` is the array size.  Host ops carry (array, mode, off, bytes).
    """
    state = {}  # array -> "H" (host newer), "D" (device newer), "B" (both valid)
    out = []
    for j, op in enumerate(trace):
        if op[0] == "launch":
            reads = {}
            for arr, mode in op[2]:
                reads[arr] = reads.get(arr, False) or mode in ("R", "RW")
            for arr, rd in reads.items():
                st = state.get(arr, "D")
                if st == "H" and rd:
                    out.append(("H2D", arr, nbytes[arr], j))
                    st = "B"
                writes = any(a == arr and m != "R" for a, m in op[2])
                state[arr] = "D" if writes else st
        elif op[0] == "host":
            arr, mode, off, nb = op[1], op[2], op[3], op[4]
            whole = off == 0 and nb == nbytes[arr]
            if not has_host[arr]:
                out.append(("H2D" if mode == "W" else "D2H", arr, nb, j))
                continue
            st = state.get(arr, "D")
            if mode == "R":
                if st == "D":
                    out.append(("D2H", arr, nb, j))
                    if whole:
                        state[arr] = "B"
            else:
                if st == "D" and not whole:
                    out.append(("D2H", arr, nbytes[arr], j))
                state[arr] = "H"
    return out
