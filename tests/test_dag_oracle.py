"""Pins for the brute-force DAG oracle (oracle/dag.py), no GPU.

* Appendix-A DAGs hand-derived from the paper's figures (tests/golden/).
* Exhaustive tiny traces: every edge is a conflict, and the transitive
  closure of the edges equals the closure of all pairwise conflicts between
  active vertices (no missing and no spurious ordering) -- PAPER.md L528-530
  ("written as if it were run sequentially").
"""
import itertools

import pytest

from oracle import dag
from golden_io import all_cases

CASES = all_cases()


@pytest.mark.parametrize("name,case", CASES, ids=[c[0] for c in CASES])
def test_golden(name, case):
    res = dag.build_dag(case["trace"])
    got_v = [(v[0], v[3] if v[2] == "kernel" else "host:" + v[3], v[4]) for v in res.vertices]
    assert got_v == case["vertices"]
    assert res.edges == case["edges"]
    if case["waits"] is not None:
        assert len(res.waits) == case["waits"]


def _closure_ok(trace):
    res = dag.build_dag(trace)
    n = len(res.vertices)
    e = dag.edge_pairs(res)
    assert e <= res.conflicts, (trace, e - res.conflicts)
    assert dag.closure(n, e) == dag.closure(n, res.conflicts), trace
    return res


OPS = []
for arrs in [("X",), ("Y",), ("X", "Y")]:
    for modes in itertools.product(("R", "RW", "O"), repeat=len(arrs)):
        OPS.append(("launch", "k", list(zip(arrs, modes))))
for arr in ("X", "Y"):
    for m in ("R", "W"):
        OPS.append(("host", arr, m, 0, 4))


def test_exhaustive_small_traces():
    """All traces of length <= 4 over 2 arrays (launch R/RW/O, host R/W)."""
    count = 0
    for length in range(1, 5):
        for tr in itertools.product(OPS, repeat=length):
            _closure_ok(list(tr))
            count += 1
    assert count > 10000


def test_random_long_traces():
    import random
    rng = random.Random(7)
    arrays = ["A", "B", "C", "D", "E"]
    for _ in range(200):
        tr = []
        for _ in range(rng.randint(5, 60)):
            r = rng.random()
            if r < 0.8:
                k = rng.randint(1, 4)
                tr.append(("launch", "k", [(rng.choice(arrays), rng.choice(["R", "R", "RW", "O"]))
                                           for _ in range(k)]))
            elif r < 0.97:
                tr.append(("host", rng.choice(arrays), rng.choice("RW"), 0, 4))
            else:
                tr.append(("sync",))
        _closure_ok(tr)


def test_readonly_siblings_run_concurrently():
    """L417-419: two kernels reading the same read-only array get different streams."""
    res = dag.build_dag([("launch", "a", [("X", "R"), ("Y", "O")]),
                         ("launch", "b", [("X", "R"), ("Z", "O")])])
    assert res.edges == set()
    assert res.vertices[0][4] != res.vertices[1][4]


def test_nonconflicting_host_access_not_recorded():
    """L512-516: accesses with no dependency on active GPU work are not vertices."""
    res = dag.build_dag([("launch", "a", [("X", "R"), ("Y", "O")]),
                         ("host", "X", "R", 0, 4),
                         ("host", "Z", "W", 0, 4)])
    assert len(res.vertices) == 1


def test_host_write_after_gpu_read_waits_for_reader():
    """Reading D6: host write waits on active readers since the last writer."""
    res = dag.build_dag([("launch", "a", [("X", "R"), ("Y", "O")]),
                         ("host", "X", "W", 0, 4)])
    assert res.edges == {(0, 1, "X")}


def test_empty_dependency_set_adds_no_edges():
    """L412-414: once every argument of K1 was overwritten, K1 adds no edges."""
    res = dag.build_dag([("launch", "k1", [("X", "O")]),
                         ("launch", "k2", [("X", "O")]),
                         ("launch", "k3", [("X", "R")])])
    assert res.edges == {(0, 1, "X"), (1, 2, "X")}


def test_transfer_oracle_counts():
    nb = {"x": 40, "y": 40, "z": 8}
    hh = {"x": True, "y": True, "z": True}
    tr = [("host", "x", "W", 0, 40),
          ("launch", "k", [("x", "R"), ("y", "O")]),
          ("launch", "k", [("x", "R"), ("z", "RW")]),
          ("host", "y", "R", 0, 40),
          ("host", "y", "R", 0, 40),
          ("host", "z", "R", 0, 4)]
    got = dag.transfers(tr, hh, nb)
    # x pulled once; y read whole once (then both valid); z range read
    assert got == [("H2D", "x", 40, 1), ("D2H", "y", 40, 3), ("D2H", "z", 4, 5)]
