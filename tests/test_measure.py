"""Host-side measurement helpers (paper_2012_09646_b200/measure.py): the
critical-path rooflines, the Fig. 9 contention-free estimate
 and the §V-F overlap metrics (L1272-1283), on hand
examples whose answers are fixed by the definitions."""
import pytest

from paper_2012_09646_b200 import measure as M


def test_critical_path_diamond_and_chain():
    # 0 -> 1 -> 3, 0 -> 2 -> 3 ; weights 1, 5, 2, 1 -> 0,1,3 = 7
    assert M.critical_path(4, [(0, 1), (0, 2), (1, 3), (2, 3)], [1, 5, 2, 1]) == 7
    assert M.critical_path(3, [], [1, 2, 3]) == 3           # independent: the max
    assert M.critical_path(3, [(0, 1), (1, 2)], [1, 2, 3]) == 6  # chain: the sum


def test_dag_rooflines_fig4_vec():
    """VEC (Fig. 4): two squares feed the reduction, which feeds the host read.
    R_cp = one square + the reduction; R_work = all three."""
    verts = [(0, "kernel", "square", 0), (1, "kernel", "square", 1), (2, "kernel", "reduce", 0),
             (3, "host", "z", -1)]
    edges = {(0, 2, "x1"), (1, 2, "y1"), (2, 3, "z")}
    cp, work = M.dag_rooflines(verts, edges, [8e9, 8e9, 8e9], 1000.0)
    assert cp == pytest.approx(16.0) and work == pytest.approx(24.0)
    cp, work = M.dag_rooflines(verts, edges, [8e9, 8e9, 8e9], 1000.0, [20.0, 1.0, 1.0])
    assert cp == pytest.approx(28.0) and work == pytest.approx(24.0)  # max(24 HBM, 22 floor)


def test_dag_rooflines_bs_golden_independent_branches():
    """B&S (10 independent kernels, Fig. 6): R_cp is ONE kernel, R_work all ten."""
    verts = [(i, "kernel", "bs", i) for i in range(10)] + [(10 + i, "host", f"c{i}", -1) for i in range(10)]
    edges = {(i, 10 + i, f"c{i}") for i in range(10)}
    cp, work = M.dag_rooflines(verts, edges, [1.6e8] * 10, 6540.8)
    assert cp == pytest.approx(1.6e8 / 6540.8e9 * 1e3)
    assert work == pytest.approx(10 * cp)


def test_contention_free_uses_host_vertex_times():
    verts = [(0, "kernel", "k", 0), (1, "host", "a", -1), (2, "kernel", "k", 0)]
    edges = {(0, 1, "a")}
    assert M.contention_free(verts, edges, [3.0, 1.0], {1: 2.0}) == 5.0


def test_overlap_metrics_hand_timeline():
    """Fig. 10-style timeline: kernels [0,4] and [2,6], a transfer [5,9].
    CT = (0 + 1)/8, TC = 1/4, CC = (2 + 2)/8, TOT = (2 + 3 + 1)/12."""
    m = M.overlap([(0, 4), (2, 6)], [(5, 9)])
    assert m["CT"] == pytest.approx(1 / 8)
    assert m["TC"] == pytest.approx(1 / 4)
    assert m["CC"] == pytest.approx(4 / 8)
    assert m["TOT"] == pytest.approx(6 / 12)
    assert m["span_ms"] == 9
    s = M.overlap([(0, 1), (2, 3)], [])
    assert s["CC"] == 0 and s["TOT"] == 0 and s["CT"] == 0
