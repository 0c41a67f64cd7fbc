"""The C++ scheduler (libdagrt.so) through its C ABI with the RECORD backend
(no GPU): DAG, stream assignment, event wiring and transfers must equal the
brute-force oracle (oracle/dag.py) bit for bit, and the Appendix-A golden DAGs.
"""
import ctypes as C
import itertools
import random

import os

import pytest

from golden_io import all_cases
from oracle import dag as odag
from paper_2012_09646_b200 import dagrt as D

MODE_TOKEN = {"R": "const ptr", "RW": "ptr", "O": "out ptr"}
CASES = all_cases()


class Replayer:
    """Replays an oracle-format trace through dagrt (record backend)."""

    def __init__(self, arrays, nbytes=64, mirrors=True, policy="parallel", prefetch=True):
        self.ctx = D.Context(backend="record", record_dag=True, policy=policy, prefetch=prefetch)
        self.bufs = {}
        self.arr = {}
        self.nbytes = {}
        for i, name in enumerate(sorted(arrays)):
            host = None
            if mirrors:
                self.bufs[name] = (C.c_char * nbytes)()
                host = C.addressof(self.bufs[name])
            self.arr[name] = self.ctx.register(name, 0x100000 * (i + 1), nbytes, host)
            self.nbytes[name] = nbytes
        self.kernels = {}
        self.scratch = (C.c_char * nbytes)()

    def kernel(self, name, modes):
        key = (name, tuple(modes))
        if key not in self.kernels:
            sig = ", ".join(MODE_TOKEN[m] for m in modes)
            self.kernels[key] = self.ctx.register_kernel(None, name, sig)
        return self.kernels[key]

    def run(self, trace):
        for op in trace:
            if op[0] == "launch":
                k = self.kernel(op[1], [m for _, m in op[2]])
                self.ctx.prepare(k, 1, 32, [self.arr[a] for a, _ in op[2]])()
            elif op[0] == "host":
                _, a, m, off, nb = op
                if m == "R":
                    self.ctx.host_read(self.arr[a], C.addressof(self.scratch), off, nb)
                else:
                    self.ctx.host_write(self.arr[a], C.addressof(self.scratch), off, nb)
            elif op[0] == "sync":
                self.ctx.sync()
        return self

    def dag(self):
        v, e = self.ctx.dag()
        return v, e

    def waits(self):
        return [t for t in self.ctx.trace() if t[0] == "wait"]

    def transfers(self):
        idx = {a.handle & 0xffffffff: n for n, a in self.arr.items()}
        out = []
        for t in self.ctx.trace():
            if t[0] in ("h2d", "d2h"):
                out.append((t[0].upper(), idx[t[2]], t[4]))
        return out


def arrays_of(trace):
    s = set()
    for op in trace:
        if op[0] == "launch":
            s |= {a for a, _ in op[2]}
        elif op[0] == "host":
            s.add(op[1])
    return s


def check_against_oracle(trace, nbytes=128, policy="parallel"):
    rp = Replayer(arrays_of(trace), nbytes, policy=policy).run(trace)
    verts, edges = rp.dag()
    o = odag.build_dag(trace, stream_policy="single" if policy == "single_stream" else "fifo")
    ov = [(v[0], v[2], v[3], v[4]) for v in o.vertices]
    gv = [(v[0], v[1], v[2], v[3]) for v in verts]
    assert gv == ov, (trace, gv, ov)
    assert edges == o.edges, (trace, edges ^ o.edges)
    gw = sorted((t[1], t[2]) for t in rp.waits())  # (stream, parent vid)
    stream_of = {v[0]: v[4] for v in o.vertices}
    ow = sorted((stream_of[c], p) for c, p in o.waits)
    assert gw == ow, trace
    ot = [(d, a, b) for d, a, b, _ in odag.transfers(trace, {a: True for a in rp.arr}, rp.nbytes)]
    assert rp.transfers() == ot, (trace, rp.transfers(), ot)
    return rp


@pytest.mark.parametrize("name,case", CASES, ids=[c[0] for c in CASES])
def test_golden_dags_through_c_abi(name, case):
    rp = check_against_oracle(case["trace"])
    verts, edges = rp.dag()
    got_v = [(v[0], v[2] if v[1] == "kernel" else "host:" + v[2], v[3]) for v in verts]
    assert got_v == case["vertices"]
    assert edges == case["edges"]
    if case["waits"] is not None:
        assert len(rp.waits()) == case["waits"]


OPS = []
for arrs in [("X",), ("Y",), ("X", "Y"), ("X", "X")]:
    for modes in itertools.product(("R", "RW", "O"), repeat=len(arrs)):
        OPS.append(("launch", "k", list(zip(arrs, modes))))
for arr in ("X", "Y"):
    for m in ("R", "W"):
        OPS.append(("host", arr, m, 0, 128))
OPS.append(("host", "X", "R", 8, 16))
OPS.append(("host", "X", "W", 8, 16))


def test_exhaustive_traces_len3():
    n = 0
    for tr in itertools.product(OPS, repeat=3):
        check_against_oracle(list(tr))
        n += 1
    assert n == len(OPS) ** 3


def test_random_traces():
    rng = random.Random(1234)
    names = list("ABCDEF")
    for _ in range(300):
        tr = []
        for _ in range(rng.randint(1, 80)):
            r = rng.random()
            if r < 0.8:
                tr.append(("launch", rng.choice(["k", "m"]),
                           [(rng.choice(names), rng.choice(["R", "R", "RW", "O"]))
                            for _ in range(rng.randint(1, 5))]))
            elif r < 0.97:
                off = rng.choice([0, 0, 8])
                nb = 128 - off if rng.random() < 0.7 else 8
                tr.append(("host", rng.choice(names), rng.choice("RW"), off, nb))
            else:
                tr.append(("sync",))
        check_against_oracle(tr)


@pytest.mark.parametrize("name,case", CASES, ids=[c[0] for c in CASES])
def test_single_stream_policy_golden(name, case):
    """The "schedule all children on a single stream" policy (L650-654):
    identical DAG (edges are policy-independent), streams and waits equal to
    the oracle's single-stream rule, and (on these DAGs) no more streams than
    the general policy."""
    rp = check_against_oracle(case["trace"], policy="single_stream")
    verts, edges = rp.dag()
    assert edges == case["edges"]
    gen = Replayer(arrays_of(case["trace"]), 128).run(case["trace"])
    assert rp.ctx.stream_count() <= gen.ctx.stream_count()


def test_single_stream_policy_random_traces():
    rng = random.Random(77)
    names = list("ABCDE")
    for _ in range(150):
        tr = []
        for _ in range(rng.randint(1, 60)):
            if rng.random() < 0.85:
                tr.append(("launch", "k", [(rng.choice(names), rng.choice(["R", "R", "RW", "O"]))
                                           for _ in range(rng.randint(1, 4))]))
            else:
                tr.append(("host", rng.choice(names), rng.choice("RW"), 0, 128))
        check_against_oracle(tr, policy="single_stream")


def test_serial_policy_has_no_edges_and_one_stream():
    tr = CASES[0][1]["trace"]
    rp = Replayer(arrays_of(tr), policy="serial").run(tr)
    verts, edges = rp.dag()
    assert edges == set()
    assert all(v[3] == -1 for v in verts)
    t = rp.ctx.trace()
    assert all(op[1] == -3 for op in t if op[0] == "launch")


def test_errors():
    ctx = D.Context(backend="record", record_dag=True)
    a = ctx.register("a", 0x1000, 256)
    with pytest.raises(D.DagrtError) as e:
        ctx.register("b", 0x1080, 256)
    assert e.value.status == D.EALIAS
    with pytest.raises(D.DagrtError) as e:
        ctx.register_kernel(None, "bad", "const ptr, wat")
    assert e.value.status == D.ESIG
    k = ctx.register_kernel(None, "k2", "const ptr, sint32")
    with pytest.raises(D.DagrtError) as e:
        ctx.prepare(k, 1, 1, [a, 3])  # ok
        D.lib().dagrt_launch(ctx._c, k.handle, D.dim3(1), D.dim3(1), 0, (D.Arg * 1)(), 1) and \
            ctx._raise(D.ESIG)
    assert e.value.status == D.ESIG
    with pytest.raises(D.DagrtError) as e:
        ctx.kernel("nope")
    assert e.value.status == D.ENOTFOUND
    ctx.unregister(a)
    with pytest.raises(D.DagrtError) as e:
        ctx.launch(k, 1, 1, a, 1)
    assert e.value.status == D.ENOTFOUND
    with pytest.raises(D.DagrtError) as e:
        ctx.host_map(ctx.register("c", 0x9000, 64), D.R)
    assert e.value.status == D.ESTATE
    b = ctx.register("b2", 0x20000, 64)
    with pytest.raises(D.DagrtError) as e:
        ctx.host_read(b, 0, 60, 8)
    assert e.value.status == D.EINVAL


def test_host_map_marks_host_newer_and_prefetches_once():
    rp = Replayer({"x", "y"})
    ctx = rp.ctx
    ctx.host_map(rp.arr["x"], D.W)
    ctx.host_unmap(rp.arr["x"])
    k = rp.kernel("k", ["R", "O"])
    ctx.prepare(k, 1, 1, [rp.arr["x"], rp.arr["y"]])()
    ctx.prepare(k, 1, 1, [rp.arr["x"], rp.arr["y"]])()
    h2d = [t for t in ctx.trace() if t[0] == "h2d"]
    assert len(h2d) == 1 and h2d[0][1] == -2  # one copy, on the copy stream
    waits = [t for t in ctx.trace() if t[0] == "wait_copy"]
    assert len(waits) >= 1


def test_all_symbols_exported():
    """Every function declared in include/dagrt.h is exported by libdagrt.so."""
    import os
    import re
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "dagrt.h")).read()
    names = set(re.findall(r"\b(dagrt_[a-z_0-9]+)\s*\(", hdr))
    L = D.lib()
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing
    assert len(names) >= 30


PRODUCT_BUILTINS = {
    "square", "reduce_diff", "bs", "bs_f32",                                          # VEC, B&S
    "blur", "sobel", "maximum", "minimum", "extend", "unsharpen", "combine",          # IMG
    "norm", "nb_mmul", "rr_mmul", "rowmax", "lse", "exp_sub", "addv", "softmax", "argmax",  # ML
    "spmv", "l2norm", "divide",                                                       # HITS
    "conv1", "pool", "conv2", "concat", "dot",                                        # DL
    "axpb", "peak_dfma", "peak_ffma",                                                 # runtime tests, peaks
}


def test_product_library_holds_only_product_kernels():
    """libdagrt.so registers exactly the product kernels; the measured variants
    come only with libdagrt_exp.so, which adds names without shadowing any
    product kernel, and a context created before it was loaded finds them."""
    import subprocess
    import sys
    code = ("from paper_2012_09646_b200 import dagrt as D\n"
            "p = [n for n, _ in D.builtins()]\n"
            "ctx = D.Context(backend='record')\n"
            "D.load_experimental()\n"
            "e = [n for n, _ in D.builtins()][len(p):]\n"
            "ctx.kernel('bs2t_o4s4b2'); ctx.kernel('spmv_merge'); ctx.kernel('conv2_ws')\n"
            "print(repr((p, e)))\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    prod, extra = eval(out.stdout.strip().splitlines()[-1])
    assert set(prod) == PRODUCT_BUILTINS and len(prod) == len(PRODUCT_BUILTINS)
    assert extra and not (set(extra) & PRODUCT_BUILTINS) and len(set(extra)) == len(extra)


@pytest.mark.parametrize("idx", range(0, len(CASES), max(1, len(CASES) // 6)))
def test_prepared_and_plain_launch_same_dag(idx):
    """dagrt_launch_prepared (one descriptor pointer per call) and dagrt_launch
    (seven arguments) are the same call: identical DAGs and traces on golden
    traces."""
    trace = CASES[idx][1]["trace"]
    out = []
    for plain in (False, True):
        rp = Replayer(arrays_of(trace), 128)
        for op in trace:
            if op[0] == "launch":
                k = rp.kernel(op[1], [m for _, m in op[2]])
                L = rp.ctx.prepare(k, 1, 32, [rp.arr[a] for a, _ in op[2]])
                if plain:
                    assert D.lib().dagrt_launch(rp.ctx._c, L.kernel.handle, L.grid, L.block, L.smem,
                                                L.args, L.n) == 0
                else:
                    L()
            else:
                rp.run([op])
        out.append((rp.dag(), rp.ctx.trace()))
    assert out[0] == out[1]


@pytest.mark.parametrize("idx", range(0, len(CASES), max(1, len(CASES) // 6)))
def test_launch_batch_same_dag(idx):
    """dagrt_launch_batch over each run of consecutive launches gives the DAG
    and trace of issuing them one by one."""
    trace = CASES[idx][1]["trace"]
    out = []
    for batched in (False, True):
        rp = Replayer(arrays_of(trace), 128)
        pending = []

        def flush():
            if pending:
                rp.ctx.batch(pending)()
                pending.clear()
        for op in trace:
            if op[0] == "launch":
                k = rp.kernel(op[1], [m for _, m in op[2]])
                L = rp.ctx.prepare(k, 1, 32, [rp.arr[a] for a, _ in op[2]])
                if batched:
                    pending.append(L)
                else:
                    L()
            else:
                flush()
                rp.run([op])
        flush()
        out.append((rp.dag(), rp.ctx.trace()))
    assert out[0] == out[1]


def test_launch_batch_stops_at_first_error():
    """dagrt_launch_batch issues the launches before a failing one and
    returns that launch's status (ESIG for an argument-count mismatch)."""
    rp = Replayer({"x", "y"}, 64)
    k = rp.kernel("k", ["R", "O"])
    good = rp.ctx.prepare(k, 1, 32, [rp.arr["x"], rp.arr["y"]])
    arr = (D.LaunchDesc * 3)()
    for i in range(3):
        C.memmove(C.byref(arr, i * C.sizeof(D.LaunchDesc)), good._dp, C.sizeof(D.LaunchDesc))
    arr[1].nargs = 1  # signature has 2
    s = D.lib().dagrt_launch_batch(rp.ctx._c, C.addressof(arr), 3)
    assert s == D.ESIG
    verts, _ = rp.dag()
    assert len(verts) == 1  # only the first launch became a vertex
    assert D.lib().dagrt_launch_batch(rp.ctx._c, None, 0) == 0


@pytest.mark.parametrize("prefetch", [True, False])
def test_copy_orders_readers_on_other_streams(prefetch):
    """A host-newer input read by two independent kernels (two streams): its
    one H2D must precede BOTH.  With the prefetcher the copy runs on the copy
    stream and both consumers wait on its event; without it the copy runs on
    the first consumer's stream and the second consumer (other stream) waits
    on the copy's event."""
    rp = Replayer({"x", "y", "z"}, prefetch=prefetch)
    ctx = rp.ctx
    ctx.host_map(rp.arr["x"], D.W)
    ctx.host_unmap(rp.arr["x"])
    k = rp.kernel("k", ["R", "O"])
    ctx.prepare(k, 1, 1, [rp.arr["x"], rp.arr["y"]])()
    ctx.prepare(k, 1, 1, [rp.arr["x"], rp.arr["z"]])()
    tr = ctx.trace()
    h2d = [t for t in tr if t[0] == "h2d"]
    assert len(h2d) == 1
    verts, _ = rp.dag()
    s0, s1 = verts[0][3], verts[1][3]
    assert s0 != s1
    waits = [t for t in tr if t[0] == "wait_copy"]
    assert sorted(t[1] for t in waits) == (sorted([s0, s1]) if prefetch else [s1])


def test_fastcall_binding_built():
    """The CPython fastcall module (pyext/dagrt_fastcall.c) is built in-tree
    and used by the per-step calls (batch, prepared reads, graph runs)."""
    assert D.fast() is not None


def test_scheduler_state_is_frontier_bounded():
    """PAPER.md L495-501 (only active computations are tracked): a long loop
    of K1 writes A, K2 reads the never-written W and A, host reads A -- the
    vertex table is dropped whenever the frontier empties, reader lists of
    read-only arrays stay bounded, and exported vertex ids stay global and
    equal to the oracle's."""
    rp = Replayer({"A", "W", "B"}, 64)
    trace = []
    for _ in range(3000):
        trace += [("launch", "k1", [("A", "O")]), ("launch", "k2", [("W", "R"), ("A", "R"), ("B", "O")]),
                  ("host", "A", "R", 0, 64), ("host", "B", "R", 0, 64)]
    rp.run(trace)
    st = rp.ctx.stats()
    assert st["table_vertices"] <= 4, st
    assert st["max_readers"] <= 33, st
    assert st["epoch_base"] > 8000, st
    verts, edges = rp.dag()
    o = odag.build_dag(trace[:40])
    assert [(v[0], v[1]) for v in verts[:len(o.vertices)]] == [(v[0], v[2]) for v in o.vertices]
    assert {e for e in edges if e[1] < len(o.vertices)} == o.edges
    assert verts[-1][0] == 4 * 3000 - 1  # global ids: 2 kernels + 2 host vertices per iteration
    # B keeps being written while W is read by every k2: the frontier never
    # empties without the host read, and readers of W are pruned as they retire
    rp2 = Replayer({"A", "W", "B"}, 64)
    tr2 = []
    for i in range(2000):
        tr2 += [("launch", "k2", [("W", "R"), ("B", "RW")])]
        if i % 10 == 9:
            tr2 += [("host", "B", "R", 0, 64)]
    rp2.run(tr2)
    assert rp2.ctx.stats()["max_readers"] <= 33


def _reg(ctx, name, nbytes, base=[0x10_0000_0000]):
    base[0] += 1 << 32
    return ctx.register(name, base[0], nbytes)


@pytest.mark.parametrize("case", [
    ("reduce_diff", 2000, 256, 0, lambda c: [_reg(c, "a", 4000), _reg(c, "b", 4000), _reg(c, "z", 8 + 8 * 2000), 1000],
     "<= 1024 CTAs"),
    ("reduce_diff", 100, 256, 0, lambda c: [_reg(c, "a", 4000), _reg(c, "b", 4000), _reg(c, "z", 100), 1000],
     "8 + 8 * grid"),
    ("square", 10, 256, 0, lambda c: [_reg(c, "a", 400), _reg(c, "b", 396), 100], "4 n bytes"),
    ("bs", 10, 256, 0, lambda c: [_reg(c, "s", 800), _reg(c, "c", 792), 100, 0.08, 0.3, 1.0, 60.0], "8 n"),
    ("blur", (1, 1), 128, 0, lambda c: [_reg(c, "i", 400), _reg(c, "o", 400), 10, 10, 7, 1.0], "diameter"),
    ("blur", (1, 1), 256, 0, lambda c: [_reg(c, "i", 400), _reg(c, "o", 400), 10, 10, 3, 1.0], "128 threads"),
    ("norm", 296, 512, 48000, lambda c: [_reg(c, "X", 4 * 1000 * 200), _reg(c, "Z", 4 * 1000 * 200),
                                         _reg(c, "st", 100), 1000, 200], "stats need"),
    ("norm", 296, 512, 1000, lambda c: [_reg(c, "X", 4 * 1000 * 200), _reg(c, "Z", 4 * 1000 * 200),
                                        _reg(c, "st", 16 + 16 * 200 + 24 * 200 * 296), 1000, 200], "shared memory"),
    ("softmax", 10, 256, 0, lambda c: [_reg(c, "x", 4 * 100 * 20), 100, 20], "C <= 16"),
    ("spmv", 10, 256, 0, lambda c: [_reg(c, "rp", 4 * 11), _reg(c, "ci", 40), _reg(c, "pl", 64), _reg(c, "x", 40),
                                    _reg(c, "y", 40), 10], "y needs"),
    ("conv2", 148, 576, 0, lambda c: [_reg(c, "p", 32 * 64 * 64), _reg(c, "w", 4608), _reg(c, "o", 64 * 32 * 32),
                                      64, 64], "shared memory"),
    ("conv2", 148, 384, 200000, lambda c: [_reg(c, "p", 32 * 64 * 64), _reg(c, "w", 4608), _reg(c, "o", 64 * 32 * 32),
                                           64, 64], "block size"),
    ("square", 10, 2048, 0, lambda c: [_reg(c, "a", 400), _reg(c, "b", 400), 100], "block of 2048"),
], ids=lambda x: x if isinstance(x, str) else None)
def test_builtin_launch_contracts_reject_bad_launches(case):
    """Every product built-in checks its launch contract before a vertex is
    made (array sizes against the shape scalars, grid / block / shared
    memory): a violation is DAGRT_EINVAL with a message, non-sticky, no
    vertex recorded -- instead of an out-of-bounds write or a hang."""
    name, grid, block, smem, args, msg = case
    ctx = D.Context(backend="record", record_dag=True)
    with pytest.raises(D.DagrtError) as e:
        ctx.launch(name, grid, block, *args(ctx), smem=smem)
    assert e.value.status == D.EINVAL and msg in str(e.value), str(e.value)
    assert ctx.dag() == ([], set())
    ok = [_reg(ctx, "a2", 400), _reg(ctx, "b2", 400), 100]
    ctx.launch("square", 1, 256, *ok)  # the context is still usable
    assert len(ctx.dag()[0]) == 1


def test_library_call_vertices_follow_the_dag_rules():
    """Library calls (dagrt_launch_library) are vertices
    like kernels: the same trace with some launches replaced by library calls
    of the same access modes gives the oracle's DAG and streams."""
    rng = random.Random(5)
    names = list("ABCD")
    for _ in range(60):
        tr = []
        for _ in range(rng.randint(1, 25)):
            if rng.random() < 0.8:
                tr.append(("launch", rng.choice(["k", "lib"]),
                           [(a, rng.choice(["R", "RW", "O"])) for a in rng.sample(names, rng.randint(1, 3))]))
            else:
                tr.append(("host", rng.choice(names), rng.choice("RW"), 0, 128))
        rp = Replayer(arrays_of(tr), 128)
        for op in tr:
            if op[0] == "launch" and op[1] == "lib":
                mode = {"R": D.R, "O": D.W, "RW": D.RW}
                rp.ctx.launch_library(lambda s: None, "lib", [rp.arr[a] for a, _ in op[2]],
                                      [mode[m] for _, m in op[2]])
            else:
                rp.run([op])
        verts, edges = rp.dag()
        o = odag.build_dag(tr)
        assert [(v[0], v[1], v[2], v[3]) for v in verts] == [(v[0], v[2], v[3], v[4]) for v in o.vertices]
        assert edges == o.edges


def test_library_call_errors():
    ctx = D.Context(backend="record", record_dag=True)
    a = ctx.register("a", 0x1000, 64)
    with pytest.raises(D.DagrtError) as e:
        ctx.launch_library(lambda s: None, "f", [a], [7])
    assert e.value.status == D.EINVAL
    ctx.launch_library(lambda s: None, "f", [a], [D.RW])
    with pytest.raises(D.DagrtError):  # a library-call name is not a launchable kernel
        ctx.launch("f", 1, 32)


def test_history_driven_launch_configuration_record():
    """f3: auto-configured launches cycle
    through the candidates `trials` times each, then settle on the fastest
    (ties -> the first: the recorder times everything as 0); histories are
    per scalar-argument key; the DAG is the one of fixed-config launches."""
    ctx = D.Context(backend="record", record_dag=True)
    a = _reg(ctx, "a", 4096)
    b = _reg(ctx, "b", 4096)
    ctx.autotune("square", [(1, 256), (2, 128), (4, 64)], trials=2)
    for _ in range(8):
        ctx.launch("square", "auto", 0, a, b, 1000)
        ctx.sync()
    chosen, ms = ctx.autotune_state("square")
    assert chosen == 0 and ms == [0.0, 0.0, 0.0]
    trace = [t for t in ctx.trace() if t[0] == "launch"]
    assert len(trace) == 8
    ctx.launch("square", "auto", 0, a, b, 500)  # another size: a fresh history
    assert ctx.autotune_state("square")[0] == -1
    verts, edges = ctx.dag()
    assert [v[2] for v in verts] == ["square"] * 9 and edges == set()
    with pytest.raises(D.DagrtError):
        ctx.launch("reduce_diff", "auto", 0, a, a, b, 10)  # no candidates registered


@pytest.mark.parametrize("prefetch", [True, False])
def test_unified_memory_arrays(prefetch):
    """Managed arrays (dagrt_array_register_managed, the UM mode of PAPER.md
    §V-C, reading D13): the DAG is the same as with mirrors.  With
    prefetch, every managed argument the host touched since its last prefetch
    -- reads and writes, pages on the host would be faulted in -- is moved by a
    prefetch on the copy stream (an h2d op in the trace), and a host read of
    device-newer data is prefetched to the host first; without prefetch no
    transfer is issued (um_fault_bytes counts the host-newer bytes left to
    page faults).  Host reads never copy (no d2h op)."""
    ctx = D.Context(backend="record", record_dag=True, prefetch=prefetch)
    bufs = [(C.c_char * 256)() for _ in range(2)]  # the recorder never touches them
    x = ctx.register_managed("x", C.addressof(bufs[0]), 256)
    y = ctx.register_managed("y", C.addressof(bufs[1]), 256)
    k = ctx.register_kernel(None, "k", "const ptr, out ptr")
    src = (C.c_char * 256)()
    ctx.host_write(x, C.addressof(src), 0, 256)  # host newer
    ctx.prepare(k, 1, 32, [x, y])()
    st = ctx.stats()
    if prefetch:  # x (host-written) and y (never prefetched since registration)
        assert [t[0] for t in ctx.trace()].count("h2d") == 2 and st["um_prefetch_bytes"] == 512
        assert st["um_fault_bytes"] == 0
    else:
        assert "h2d" not in [t[0] for t in ctx.trace()]
        assert st["um_fault_bytes"] == 256 and st["um_prefetch_bytes"] == 0
    ctx.host_read(y, C.addressof(src), 0, 256)  # device newer: prefetched to the host first (prefetch on)
    st = ctx.stats()
    assert st["um_prefetch_bytes"] == (768 if prefetch else 0)
    assert "d2h" not in [t[0] for t in ctx.trace()] and st["d2h_copies"] == 0
    v, e = ctx.dag()
    assert [t[1] for t in v] == ["kernel", "host"] and len(e) == 1
    # again: x is current on the device; y was touched by the host read
    ctx.prepare(k, 1, 32, [x, y])()
    st2 = ctx.stats()
    if prefetch:
        assert st2["um_prefetch_bytes"] == 1024
    else:
        assert st2["um_fault_bytes"] == 256
    ctx.close()
