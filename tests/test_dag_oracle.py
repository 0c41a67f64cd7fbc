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


def _simulate(trace, transfers, has_host, nbytes):
    """Two-copy machine (device array + host mirror) driven by the transfer
    oracle's copies, against a one-copy machine (plain sequential memory):
    every value a kernel or a host read observes must be the same.  Kernels
    read their read arguments whole and overwrite their written arguments
    whole with a value derived from the op index and what they read; host
    writes store the op index into their byte range."""
    import numpy as np
    one = {a: np.zeros(nbytes[a], np.int64) for a in nbytes}
    dev = {a: np.zeros(nbytes[a], np.int64) for a in nbytes}
    host = {a: np.zeros(nbytes[a], np.int64) for a in nbytes}  # mirror starts stale
    copies = {}
    for c in transfers:
        copies.setdefault(c[3], []).append(c)
    for j, op in enumerate(trace):
        for kind, arr, nb, _ in copies.get(j, []):
            if op[0] == "host" and has_host[arr]:
                off = op[3] if nb == op[4] else 0  # a range read, or the whole-array pull
                if kind == "D2H":
                    host[arr][off:off + nb] = dev[arr][off:off + nb]
            elif kind == "H2D" and op[0] == "launch":
                dev[arr][:] = host[arr]
        if op[0] == "launch":
            seen1 = [int(one[a].sum() * 31 + one[a][::7].sum()) for a, m in op[2] if m != "O"]
            seen2 = [int(dev[a].sum() * 31 + dev[a][::7].sum()) for a, m in op[2] if m != "O"]
            assert seen1 == seen2, (j, op)
            val = 1000 * (j + 1) + sum(seen1) % 997
            for a, m in op[2]:
                if m != "R":
                    one[a][:] = val
                    dev[a][:] = val
        elif op[0] == "host":
            _, arr, mode, off, nb = op
            if mode == "R":
                mine = (host[arr] if has_host[arr] else dev[arr])[off:off + nb]
                assert np.array_equal(mine, one[arr][off:off + nb]), (j, op)
            else:
                one[arr][off:off + nb] = j + 1
                (host[arr] if has_host[arr] else dev[arr])[off:off + nb] = j + 1


def test_transfer_oracle_semantics_brute_force():
    """Pins the transfer oracle (incl. its partial-write rule: a partial host
    write of a device-newer array first pulls the WHOLE array, because the
    next upload sends the whole mirror) against plain sequential memory on
    every trace of length <= 4 over one array and on random traces over
    three arrays, with and without host mirrors.  Dropping the pull, or
    pulling only the written range, fails it."""
    import itertools
    import random
    nb = {"X": 16, "Y": 16, "Z": 16}
    ops1 = [("launch", "k", [("X", m)]) for m in ("R", "RW", "O")] + \
           [("host", "X", m, off, n) for m in "RW" for off, n in ((0, 16), (4, 8), (12, 4))]
    for L in range(1, 5):
        for tr in itertools.product(ops1, repeat=L):
            tr = list(tr)
            for hh in (True, False):
                hv = {"X": hh}
                _simulate(tr, dag.transfers(tr, hv, nb), hv, nb)
    rng = random.Random(9)
    for _ in range(400):
        tr = []
        for _ in range(rng.randint(1, 30)):
            if rng.random() < 0.6:
                tr.append(("launch", "k", [(rng.choice("XYZ"), rng.choice(["R", "RW", "O"]))
                                           for _ in range(rng.randint(1, 3))]))
            else:
                off = rng.choice([0, 0, 4, 8])
                tr.append(("host", rng.choice("XYZ"), rng.choice("RW"), off, rng.choice([16 - off, 4])))
        # a kernel using the same array twice with different modes: merged (D3)
        hv = {a: rng.random() < 0.8 for a in "XYZ"}
        _simulate(tr, dag.transfers(tr, hv, nb), hv, nb)


def test_transfer_simulator_catches_a_missing_pull():
    """The brute-force check above is sharp: removing the whole-array pull
    of the partial-write rule makes it fail."""
    nb = {"X": 16}
    hv = {"X": True}
    tr = [("launch", "k", [("X", "O")]), ("host", "X", "W", 4, 4), ("launch", "k", [("X", "R")])]
    good = dag.transfers(tr, hv, nb)
    _simulate(tr, good, hv, nb)
    bad = [c for c in good if not (c[0] == "D2H" and c[3] == 1)]
    with pytest.raises(AssertionError):
        _simulate(tr, bad, hv, nb)
