"""Multi-GPU DAG placement (f2; csrc/multi.cpp, include/dagrt.h "multi-GPU
placement"; §VII) on the RECORD backend: placement by
data location and estimated migration cost, migrations as library-call
vertices ordered by the slot schedulers (cross-slot RAW / WAR / WAW), and
the validity bookkeeping.  No device work is done here; the GPU test
(tests/test_gpu_multi.py) runs the same paths on a B200."""
import numpy as np
import pytest

from paper_2012_09646_b200 import dagrt as D

N = 10_000_000  # B&S vector length (BASELINE configs[1]): 80 MB per fp64 vector
BS = (0.08, 0.30, 1.0, 60.0)


def multi(nslots=2, placement="data"):
    return D.Multi(devices=[0] * nslots, placement=placement, backend="record", record_dag=True)


def host_buf(nbytes):
    # the recorder never dereferences device or host pointers; a small real
    # buffer stands for the mirror (host writes pass it as its own source)
    return np.zeros(16, np.uint8)


def names(ctx):
    v, _ = ctx.dag()
    return [x[2] for x in v]


def test_independent_kernels_spread_over_slots_from_the_host():
    """B&S from host-newer inputs (the stream mode of the benchmark): every
    slot is equally far from the host, so the busy estimate spreads the 10
    kernels evenly, each preceded by its upload on the slot it runs on."""
    m = multi(2)
    buf = host_buf(0)
    S = [m.register(f"s{i}", 8 * N, host_ptr=buf.ctypes.data) for i in range(10)]
    Cs = [m.register(f"c{i}", 8 * N) for i in range(10)]
    placed = [m.launch("bs", 296, 256, S[i], Cs[i], N, *BS) for i in range(10)]
    assert placed == [0, 1] * 5
    st = m.stats()
    assert st["per_slot"] == [5, 5] and st["migrations_host"] == 10 and st["migrations_peer"] == 0
    for s in (0, 1):
        assert names(m.slot_context(s)) == ["upload", "bs"] * 5
    m.close()


def test_resident_inputs_stay_until_the_queue_costs_more_than_the_copy():
    """Inputs resident on slot 0: a kernel moves to slot 1 only once slot 0's
    estimated queue exceeds the peer copy of its input (80 MB over the
    same-device path at 3000 GB/s = 26.7 us, vs 24.6 us of HBM time per
    kernel): data placement migrates far fewer bytes than round-robin."""
    res = {}
    for pol in ("data", "round_robin"):
        m = multi(2, pol)
        S = [m.register(f"s{i}", 8 * N, home=0, dev_ptr=(1 << 40) + i * (1 << 30)) for i in range(10)]
        Cs = [m.register(f"c{i}", 8 * N) for i in range(10)]
        res[pol] = ([m.launch("bs", 296, 256, S[i], Cs[i], N, *BS) for i in range(10)], m.stats())
        m.close()
    placed, st = res["data"]
    assert placed[0] == 0 and placed[1] == 0  # the first ones stay with their data
    assert st["migrations_peer"] == placed.count(1)
    assert res["round_robin"][1]["migrations_peer"] == 5
    assert st["bytes_peer"] <= res["round_robin"][1]["bytes_peer"]


def test_cross_slot_chain_migrates_and_orders():
    """VEC across slots: x1 = x^2 on slot 1 (x resident on slot 0), y1 = y^2 on
    slot 0, z = sum(x1 - y1) on slot 0.  Slot 1: migrate_pre -> migrate_in ->
    square; slot 0: migrate_out reads x after nothing, and the reduction waits
    for x1 to come back (migrate_in on slot 0 after slot 1's square)."""
    m = multi(2)
    n = 1000
    x = m.register("x", 4 * n, home=0, dev_ptr=1 << 40)
    y = m.register("y", 4 * n, home=0, dev_ptr=(1 << 40) + (1 << 20))
    x1, y1, z = m.register("x1", 4 * n), m.register("y1", 4 * n), m.register("z", 128)
    assert m.launch("square", 8, 256, x, x1, n, slot=1) == 1
    assert m.launch("square", 8, 256, y, y1, n, slot=0) == 0
    assert m.launch("reduce_diff", 8, 256, x1, y1, z, n, slot=0) == 0
    c0, c1 = m.slot_context(0), m.slot_context(1)
    v1, e1 = c1.dag()
    assert [x[2] for x in v1] == ["migrate_pre", "migrate_in", "square", "migrate_out"]
    ids1 = {x[2]: x[0] for x in v1}
    pairs1 = {(p, c) for p, c, _ in e1}
    assert (ids1["migrate_pre"], ids1["migrate_in"]) in pairs1      # WAW on the replica
    assert (ids1["migrate_in"], ids1["square"]) in pairs1           # RAW: x arrived
    assert (ids1["square"], ids1["migrate_out"]) in pairs1          # x1 leaves after it is written
    v0, e0 = c0.dag()
    assert [x[2] for x in v0] == ["migrate_out", "square", "migrate_pre", "migrate_in", "reduce_diff"]
    ids0 = {x[2]: x[0] for x in v0}
    pairs0 = {(p, c) for p, c, _ in e0}
    assert (ids0["migrate_in"], ids0["reduce_diff"]) in pairs0      # RAW on x1
    assert (ids0["square"], ids0["reduce_diff"]) in pairs0          # RAW on y1
    st = m.stats()
    assert st["migrations_peer"] == 2 and st["bytes_peer"] == 8 * n
    m.close()


def test_writer_waits_for_the_outgoing_copy():
    """WAR across slots: slot 1 reads x (copied out of slot 0), then slot 0
    overwrites x: in slot 0's DAG the writer depends on migrate_out."""
    m = multi(2)
    n = 1000
    x = m.register("x", 4 * n, home=0, dev_ptr=1 << 40)
    w = m.register("w", 4 * n, home=0, dev_ptr=(1 << 40) + (1 << 20))
    x1 = m.register("x1", 4 * n)
    m.launch("square", 8, 256, x, x1, n, slot=1)
    m.launch("square", 8, 256, w, x, n, slot=0)  # overwrites x on slot 0
    v0, e0 = m.slot_context(0).dag()
    ids0 = {x[2]: x[0] for x in v0}
    assert (ids0["migrate_out"], ids0["square"]) in {(p, c) for p, c, _ in e0}
    m.close()


def test_reads_follow_the_current_copy():
    """After a write on slot 1 the only current copy is there: the host read
    goes through slot 1's scheduler (a host vertex in its DAG), and a later
    reader on slot 0 migrates it back; a reader of data current everywhere
    migrates nothing."""
    m = multi(2)
    n = 1000
    x = m.register("x", 4 * n, home=0, dev_ptr=1 << 40)
    x1 = m.register("x1", 4 * n)
    x2 = m.register("x2", 4 * n)
    m.launch("square", 8, 256, x, x1, n, slot=1)
    out = np.zeros(n, np.float32)
    m.read(x1, out.ctypes.data)
    v1, _ = m.slot_context(1).dag()
    assert any(t[1] == "host" for t in v1)
    before = m.stats()["migrations_peer"]
    m.launch("square", 8, 256, x1, x2, n, slot=0)
    assert m.stats()["migrations_peer"] == before + 1
    m.launch("square", 8, 256, x, x2, n, slot=1)  # x is current on both slots now
    assert m.stats()["migrations_peer"] == before + 1
    m.close()


def test_errors():
    m = multi(2)
    x = m.register("x", 64, home=0, dev_ptr=1 << 40)
    y = m.register("y", 64)
    with pytest.raises(D.DagrtError) as e:
        m.launch("square", 1, 32, x, y, slot=0)
    assert e.value.status == D.ESIG
    with pytest.raises(D.DagrtError):
        m.launch("square", 1, 32, x, y, 16, slot=2)
    with pytest.raises(D.DagrtError):
        m.launch("no_such_kernel", 1, 32, x, y, 16)
    with pytest.raises(D.DagrtError) as e:
        m.read(y, np.zeros(16, np.float32).ctypes.data)  # never written anywhere
    assert e.value.status == D.ESTATE
    with pytest.raises(D.DagrtError):
        m.register("bad", 64, home=5)
    m.close()
