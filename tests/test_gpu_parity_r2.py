"""GPU parity cases added in round 2 (VERDICT r1 "Make parity green"):

* every benchmark under every scheduling policy (serial-sync, PAPER.md
  L559-569 -- the baseline every speedup divides by; the graph cache;
  the hand-written CUDA graph) against the fp64 oracle, both modes;
* NORM on wide-range integer X (exact 128-bit sums);
* DL at 4096^2 (about 14 conv2 tiles per CTA, so every TMA stage and
  mbarrier phase of the product kernel is reused) element-wise, and at the
  full 16384^2 size c2x/c2y strips element-wise plus r against the oracle's r;
* B&S at the limits S << K and S >> K;
* the graph cache's ordering across a flush with a vertex still active.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import bs as obs
from oracle import dl as odl
from oracle import ml as oml
from paper_2012_09646_b200 import dagrt as D
from paper_2012_09646_b200.programs import (BlackScholes, DeepLearning, Hits, Images, MLEnsemble,
                                            Vec)

from oracle_checks import assert_close, check, red

pytestmark = pytest.mark.gpu

SMALL = {
    "vec": lambda c, m: Vec(c, n=100_003, mode=m),
    "bs": lambda c, m: BlackScholes(c, n=40_009, mode=m),
    "bs_f32": lambda c, m: BlackScholes(c, n=40_009, mode=m, dtype="f32"),
    "img": lambda c, m: Images(c, h=300, w=517, mode=m),
    "ml": lambda c, m: MLEnsemble(c, n=20_011, mode=m),
    "hits": lambda c, m: Hits(c, n=50_000, e=150_000, iters=3, mode=m),
    "dl": lambda c, m: DeepLearning(c, h=515, w=517, mode=m),
}


@pytest.mark.parametrize("bench", list(SMALL))
@pytest.mark.parametrize("mode", ["resident", "stream"])
@pytest.mark.parametrize("policy", ["serial", "graph_cache", "single_stream"])
def test_policy_outputs_match_oracle(bench, mode, policy):
    """The same program under another policy computes the oracle's results,
    run three times (the graph cache replays from the third run on)."""
    kw = {"graph_cache": True} if policy == "graph_cache" else {"policy": policy}
    c = D.Context(device=0, **kw)
    p = SMALL[bench](c, mode)
    p.load_inputs(2)
    for _ in range(3):
        if bench == "hits":  # iterations restart from 1/sqrt(N) each run
            p.restart()
        p.run()
    c.sync()
    check(p, 2)
    if policy == "graph_cache":
        st = c.stats()
        assert st["graph_replays"] >= 1, st
    del p
    c.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("bench", list(SMALL))
@pytest.mark.parametrize("policy,prefetch", [("parallel", True), ("parallel", False), ("serial", False)])
def test_unified_memory_mode_matches_oracle(bench, policy, prefetch):
    """UM mode (managed arrays, §V-C): inputs'
    pages moved to the host before each run, then prefetched by the runtime
    (cudaMemPrefetchAsync) or faulted in by the kernels; the host reads the
    sinks in place.  Three runs, the oracle's results each time."""
    c = D.Context(device=0, policy=policy, prefetch=prefetch)
    p = SMALL[bench](c, "um")
    p.load_inputs(3)
    c.stats_reset()
    for _ in range(3):
        p.restart()
        p.run()
        c.sync()
        check(p, 3)
    st = c.stats()
    if prefetch:
        assert st["um_prefetch_bytes"] > 0 and st["um_fault_bytes"] == 0, st
    else:
        assert st["um_fault_bytes"] > 0 and st["um_prefetch_bytes"] == 0, st
    assert st["d2h_copies"] == 0, st  # the host reads managed memory in place
    del p
    c.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("bench", list(SMALL))
@pytest.mark.parametrize("mode", ["resident", "stream"])
def test_hand_written_graph_matches_oracle(bench, mode):
    c = D.Context(device=0)
    p = SMALL[bench](c, mode)
    p.load_inputs(1)
    g = p.graph()
    if mode == "stream":
        p.begin_run()  # host-newer inputs; the graph's H2D nodes upload them
    g.run()
    torch.cuda.synchronize()
    check(p, 1)
    del p, g
    c.close()
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ NORM
@pytest.mark.parametrize("n,lo,hi", [(100_003, -(1 << 20), 1 << 20),
                                     (40_000, -(1 << 31), (1 << 31) - 1),
                                     (7, 0, 2)])
def test_ml_norm_wide_range(n, lo, hi):
    """X ~ U{lo..hi}: the sum of squares exceeds 64 bits for the full int32
    range (40k rows x 2^62); NORM's statistics must still be exact."""
    c = D.Context(device=0)
    p = MLEnsemble(c, n=n)
    p.load_inputs(0)
    rng = np.random.default_rng(n)
    X = rng.integers(lo, hi, size=(n, p.f), endpoint=True).astype(np.int32)
    p.t["X"].copy_(torch.from_numpy(X.ravel()))
    p.settle()
    p.run()
    c.sync()
    mu, sd = oml.norm_stats(X)
    st = p.t["stats"][16:16 + 16 * p.f].view(torch.float64).cpu().numpy()
    assert np.allclose(st[:p.f], mu, rtol=1e-12, atol=1e-9 * max(1, abs(lo), hi))
    assert np.allclose(1.0 / st[p.f:], sd, rtol=1e-12)
    Z = p.t["Z"].cpu().numpy().reshape(n, p.f)
    assert_close(Z, oml.apply_norm(X, mu, sd), "Z")
    if n > 100:
        pr = {k: v.astype(np.float64) for k, v in p.params.items()}
        r2 = oml.softmax(oml.addv(oml.mmul(oml.apply_norm(X, mu, sd), pr["W"]), pr["b"]))
        assert_close(p.t["r2"].cpu().numpy().reshape(n, p.c), r2, "r2")
    c.close()


# ------------------------------------------------------------------ DL
def test_dl_4096_elementwise():
    """4096^2: 2,048 conv2 tiles over 148 CTAs x 3 consumer groups -> every
    group reuses its TMA stage and flips its mbarrier phase several times."""
    c = D.Context(device=0)
    p = DeepLearning(c, h=4096, w=4096)
    p.load_inputs(0)
    p.run()
    c.sync()
    check(p, 0)
    del p
    c.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kernel", ["conv2_ws", "conv2_ws6", "conv2_ws6s8", "conv2_ws6b3", "conv2_ws5s8b3",
                                    "conv2_rows", "conv2_rows_s4", "conv2_rows_r20", "conv2_h", "conv2_h_s8",
                                    "conv2_h_b4", "conv2_h_s16", "conv2_h_s24", "conv2_h_s12b4", "conv2_h_s24b4",
                                    "conv2_hs", "conv2_hs_r12", "conv2_hs_s8", "conv2_hs_s16", "conv2_h_r16",
                                    "conv2_h_r20", "conv2_h_r24"])
@pytest.mark.parametrize("h,w", [(19, 23), (515, 517), (1030, 2050), (4096, 4096)])
def test_conv2_ws_matches_oracle(exp, h, w, kernel):
    """The warp-specialised conv2 (A_lo in TMEM; csrc/kernels_conv2.cu) against
    the oracle's conv on the pooled input, from one tile to ~14 tiles per CTA
    (every stage / TMEM buffer / barrier phase reused many times), ragged
    output rows (W3 not a multiple of 128)."""
    from paper_2012_09646_b200.programs.hits_dl import conv2_ws_launch
    threads, smem = conv2_ws_launch(kernel)
    c = D.Context(device=0)
    p = DeepLearning(c, h=h, w=w)
    p.load_inputs(1)
    p.run()
    c.sync()
    (h1, w1s), (h2, w2s), (h3, w3s) = p.shapes
    out = torch.full((h3 * w3s * 16,), -1.0, device="cuda")
    torch.cuda.synchronize()
    o_arr = c.register_tensor("c2ws", out)
    for _ in range(2):
        c.launch(kernel, 148, threads, p.a["px"], p.a["w2"], o_arr, h2, w2s, smem=smem)
    c.sync()
    spec = synth.spec_dl(h, w)
    w2 = synth.draw(p.seed, "w2", spec["w2"]).reshape(16, 3, 3, 8)
    px = p.t["px"][:h2 * w2s * 8].cpu().numpy().reshape(h2, w2s, 8)
    ref = odl.conv3x3s2(px, w2)
    assert_close(out.cpu().numpy().reshape(h3, w3s, 16), ref, "conv2_ws")
    del p
    c.close()
    torch.cuda.empty_cache()


def _c2_strip(seed, spec, name, h, w, w1, w2, P0, P1):
    """Oracle conv2 output rows [P0, P1) of a full-size branch, from input
    rows [8*P0 - 8, 8*P1 + 8) (aligned to 8, so every stride lines up; the
    strip's artificial zero border only reaches the discarded first row)."""
    xa, xb = max(0, 8 * P0 - 8), min(h, 8 * P1 + 8)
    idx = np.arange(xa * w, xb * w, dtype=np.uint64)
    x = synth.draw(seed, name, spec[name], idx).reshape(xb - xa, w)
    c2 = odl.conv3x3s2(odl.pool2x2(odl.conv3x3s2(x, w1)), w2)
    off = (P0 - xa // 8)
    return c2[off:off + (P1 - P0)]


def test_dl_full_size_strips_and_r():
    """2 x 16384^2 (BASELINE configs[4], bench launch configuration): c2x and
    c2y element-wise on strips spread over the image (first/last rows, every
    CTA's interleaved tiles), and r = z . wd against the oracle's r computed
    from the oracle's own c2 over the whole image (strip by strip)."""
    h = w = 16384
    c = D.Context(device=0)
    p = DeepLearning(c, h=h, w=w)
    p.load_inputs(0)
    p.run()
    c.sync()
    spec = synth.spec_dl(h, w)
    w1 = synth.draw(p.seed, "w1", spec["w1"]).reshape(8, 3, 3, 1)
    w2 = synth.draw(p.seed, "w2", spec["w2"]).reshape(16, 3, 3, 8)
    wd = synth.draw(p.seed, "wd", spec["wd"]).astype(np.float64)
    (_, _), (_, _), (h3, w3s) = p.shapes
    half = h3 * w3s * 16
    r_o = 0.0
    strip = 256
    checked = {0, h3 // strip // 2, h3 // strip - 1}
    for bi, name in enumerate(("x", "y")):
        for s0 in range(0, h3, strip):
            s1 = min(h3, s0 + strip)
            ref = _c2_strip(p.seed, spec, name, h, w, w1, w2, s0, s1)
            lo = bi * half + s0 * w3s * 16
            r_o += float(np.dot(ref.ravel(), wd[lo:lo + ref.size]))
            if s0 // strip in checked:
                got = p.t[f"c2{name}"][s0 * w3s * 16:s1 * w3s * 16].cpu().numpy()
                assert_close(got, ref.ravel(), (name, s0))
    assert abs(red(p.t["r"]) - r_o) <= 1e-3 * abs(r_o), (red(p.t["r"]), r_o)
    del p
    c.close()
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ B&S limits
@pytest.mark.parametrize("svals", [[1e-3, 1.0, 600.0, 1e6], [59.999, 60.0, 60.001, 1e-300, 5e5]])
def test_bs_limits(svals):
    """S << K (C -> 0: the 1e-12 absolute term) and S >> K (C -> S - K e^-RT)
    through the product kernel's table-driven log/exp, ragged length."""
    n = 4 * 1031 + 3
    c = D.Context(device=0)
    p = BlackScholes(c, n=n, nvec=1)
    s = np.resize(np.asarray(svals, np.float64), n)
    p.t["s0"].copy_(torch.from_numpy(s))
    p.settle()
    p.run()
    c.sync()
    ref = obs.call(s)
    out = p.t["c0"].cpu().numpy()
    err = np.abs(out - ref) - (1e-10 * np.abs(ref) + 1e-12)
    assert np.all(err <= 0), (float(err.max()), s[np.argmax(err)])
    c.close()


@pytest.mark.parametrize("kernel", ["bs", "bs2_p3w2b2", "bs2_p2w4b2", "bs2t_o4s4b2", "bs2t_o6s3b2", "bs3_o6s4b2",
                                    "bs3_o4s8b2", "bs2l_o6s3b2", "bs2l_o4s3b3", "bs2m_o6s3b2", "bs2m_o4s3b3",
                                    "bs2m_o6s3b3", "bs2m_o8s2b2", "bs2m_o4s4b2", "bs3_o6s4b2l", "bs3_o4s6b3l"])
def test_bs_kernels_limits_and_range(exp, kernel):
    """Every B&S pricing kernel on the limit values plus a dense S sweep over
    [1e-3, 1e4] (log-spaced): deep out of / in the money, d ~ 0, the exp's
    underflow clamp; 1e-10 relative + 1e-12 absolute."""
    n = 200_003
    s = np.concatenate([np.array([1e-3, 1.0, 600.0, 1e6, 59.999, 60.0, 60.001, 1e-300, 5e5]),
                        np.logspace(-3, 4, n - 9)])
    ts = torch.from_numpy(s).cuda()
    tc = torch.full_like(ts, -1.0)
    c = D.Context(device=0)
    torch.cuda.synchronize()
    S = c.register_tensor("s", ts)
    Cc = c.register_tensor("c", tc)
    from paper_2012_09646_b200.programs.vec_bs import bs_launch
    block, smem = bs_launch(kernel)
    c.launch(kernel, 37, block, S, Cc, n, obs.R, obs.V, obs.T, obs.K, smem=smem)
    c.sync()
    ref = obs.call(s)
    out = tc.cpu().numpy()
    err = np.abs(out - ref) - (1e-10 * np.abs(ref) + 1e-12)
    assert np.all(err <= 0), (float(err.max()), s[np.argmax(err)], out[np.argmax(err)], ref[np.argmax(err)])
    c.close()


# ------------------------------------------------------------------ graph cache ordering
def test_graph_cache_orders_same_stream_work_across_flush():
    """K1 writes A, K2 writes B, host reads B (K1 stays active),
    loop.  In the next run K1' (child of the still-active K1, same stream, no
    event wait) must not overlap K1 when it replays inside a graph.  A is
    incremented by each K1: after R runs every element equals R."""
    c = D.Context(device=0, graph_cache=True)
    n = 1 << 22
    A = torch.zeros(n, device="cuda")
    B = torch.zeros(n, device="cuda")
    torch.cuda.synchronize()
    a = c.register_tensor("A", A)
    b = c.register_tensor("B", B)
    import ctypes as C
    buf = (C.c_float * 1)()
    runs = 12
    for _ in range(runs):
        for _ in range(8):  # a long chain on A's stream keeps K1 in flight
            c.launch("axpb", 4 * 148, 256, a, n, 1.0, 0.125)
        c.launch("axpb", 148, 256, b, n, 1.0, 1.0)
        c.host_read(b, C.addressof(buf), 0, 4)
    c.sync()
    assert torch.all(A == runs).item(), float((A - runs).abs().max())
    assert torch.all(B == runs).item()
    st = c.stats()
    assert st["graph_replays"] >= runs - 3, st
    c.close()


@pytest.mark.parametrize("events", ["learn", "vertex", "tail"])
def test_graph_cache_host_reads_of_mid_stream_vertices(events, monkeypatch):
    """f1 event-record nodes (DAGRT_F1_EVENTS): per run K1 A += 1, K2 C = A^2
    (K2 follows K1 on its stream, so K1 is not the stream's tail), K3 B += 1
    on another stream; the host reads B (flushes the batch), then A (waits
    on K1's event from OUTSIDE the batch: an escaped record, given its own
    node in "learn" mode after the eager first issue), then C.  Every read
    sees run r's values in all three modes."""
    monkeypatch.setenv("DAGRT_F1_EVENTS", events)
    c = D.Context(device=0, graph_cache=True)
    n = 1 << 20
    A = torch.zeros(n, device="cuda")
    B = torch.zeros(n, device="cuda")
    Cc = torch.zeros(n, device="cuda")
    torch.cuda.synchronize()
    a, b, cc = (c.register_tensor(k, t) for k, t in (("A", A), ("B", B), ("C", Cc)))
    import ctypes as C
    buf = (C.c_float * 4)()
    for r in range(1, 9):
        c.launch("axpb", 148, 256, a, n, 1.0, 1.0)
        c.launch("square", 148, 256, a, cc, n)
        c.launch("axpb", 148, 256, b, n, 1.0, 1.0)
        c.host_read(b, C.addressof(buf), 4 * (n - 4), 16)
        assert list(buf) == [r] * 4
        c.host_read(a, C.addressof(buf), 0, 16)
        assert list(buf) == [r] * 4
        c.host_read(cc, C.addressof(buf), 4 * (n // 2), 16)
        assert list(buf) == [r * r] * 4
    c.sync()
    assert c.stats()["graph_replays"] >= 4
    c.close()


# ------------------------------------------------------------------ library-call vertices
def test_library_call_vertex_on_the_gpu():
    """A library call (torch.matmul on the stream the scheduler picked,
    PAPER.md L516-519) between two kernels: X1 = X^2 (kernel), Y = X1 W
    (library), Y1 = Y^2 (kernel); the host reads Y1.  Results equal the fp64
    reference and the DAG is the chain the access modes imply."""
    n, f = 4096, 64
    c = D.Context(device=0, record_dag=True)
    X = torch.rand(n * f, device="cuda")
    X1 = torch.empty_like(X)
    W = torch.rand(f, f, device="cuda")
    Y = torch.empty(n * f, device="cuda")
    Y1 = torch.empty_like(Y)
    torch.cuda.synchronize()
    a = {k: c.register_tensor(k, t) for k, t in (("X", X), ("X1", X1), ("W", W), ("Y", Y), ("Y1", Y1))}
    c.launch("square", 64, 256, a["X"], a["X1"], n * f)

    def mm(stream):
        with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
            torch.matmul(X1.view(n, f), W, out=Y.view(n, f))
    c.launch_library(mm, "matmul", [a["X1"], a["W"], a["Y"]], [D.R, D.R, D.W])
    c.launch("square", 64, 256, a["Y"], a["Y1"], n * f)
    import ctypes as C
    buf = (C.c_float * 1)()
    c.host_read(a["Y1"], C.addressof(buf), 0, 4)
    c.sync()
    ref = ((X.double().view(n, f) ** 2) @ W.double()) ** 2
    assert torch.allclose(Y1.view(n, f).double(), ref, rtol=2e-3)
    verts, edges = c.dag()
    assert [v[2] for v in verts[:3]] == ["square", "matmul", "square"]
    assert {(p, ch) for p, ch, _ in edges} == {(0, 1), (1, 2), (2, 3)}
    c.close()


# ------------------------------------------------------------------ f3: history-driven launch configuration
def test_autotune_picks_the_faster_configuration():
    """Auto-configured B&S launches explore a 2-CTA and a full-GPU grid, then
    keep the faster (the full one, ~100x); prices equal the oracle's under
    every configuration tried."""
    n = 2_000_003
    c = D.Context(device=0)
    p = BlackScholes(c, n=n, nvec=1)
    p.load_inputs(0)
    c.autotune("bs", [(2, 256), (296, 256)], trials=2)
    for _ in range(6):
        c.launch("bs", "auto", 0, p.a["s0"], p.a["c0"], n, obs.R, obs.V, obs.T, obs.K)
        c.sync()
    chosen, ms = c.autotune_state("bs")
    assert chosen == 1 and ms[0] > 5 * ms[1], (chosen, ms)
    from oracle_checks import check_bs
    check_bs(p, p.seed)
    c.close()


# ------------------------------------------------------------------ L2 norm
@pytest.mark.parametrize("n,offset,grid", [(5_000_003, 0, 592), (5_000_003, 1, 592), (20_000_000, 0, 592),
                                           (1_000_000, 0, 592), (4099, 0, 17), (1, 0, 1), (0, 0, 3),
                                           (3_000_001, 2, 1024)])
def test_l2norm_matches_oracle(n, offset, grid):
    """The product l2norm: float4 streams with a scalar tail, the unaligned
    (scalar) path, tiny and empty vectors, several grids; ||v|| vs the fp64
    sum (SUM node of the HITS DAG, reading R-HITS), 1e-6 relative (fp32
    squares per float4)."""
    c = D.Context(device=0)
    base = torch.rand(n + offset + 4, device="cuda") * 2 - 1
    v = base[offset:offset + n]
    out = torch.zeros(8 + 8 * 1024, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    V = c.register_tensor("v", v)
    O = c.register_tensor("o", out)
    c.launch("l2norm", grid, 256, V, O, n)
    c.sync()
    got = float(out[:4].view(torch.float32)[0])
    ref = float(np.sqrt(np.sum(v.double().cpu().numpy() ** 2)))
    assert abs(got - ref) <= 1e-6 * max(ref, 1e-30), (got, ref)
    # reusable: the arrival counter is reset by the last CTA
    c.launch("l2norm", grid, 256, V, O, n)
    c.sync()
    assert float(out[:4].view(torch.float32)[0]) == got
    c.close()


# ------------------------------------------------------------------ IMG stencils, edge shapes
@pytest.mark.parametrize("h,w,offset", [(1, 1, 0), (2, 3, 1), (3, 5, 0), (7, 4099, 1), (130, 1030, 0),
                                        (64, 1000, 0), (65, 513, 3), (5, 4096, 0)])
def test_img_stencils_edge_shapes(h, w, offset):
    """The product blur (d = 1, 3, 5) and sobel (cp.async row ring, PF rows
    ahead; img_stencil.cuh) on images shorter than the ring, narrower than a
    tile, with W % 4 != 0 and misaligned bases (the 4-byte copy path), and
    a ragged last tile; against the fp64 oracle (zero padding), fp32 1e-4
    relative + 1e-6 absolute (reading R-IMG)."""
    from oracle import img as oimg
    c = D.Context(device=0)
    rng = np.random.default_rng(h * 7919 + w)
    img = rng.random((h, w))
    base = torch.zeros(h * w + 8, device="cuda")
    x = base[offset:offset + h * w]
    x.copy_(torch.from_numpy(img.astype(np.float32).ravel()))
    y = torch.full((h * w,), -7.0, device="cuda")
    torch.cuda.synchronize()
    X = c.register_tensor("x", x)
    Y = c.register_tensor("y", y)
    grid = (max(1, -(-w // 512)), max(1, -(-h // 64)))
    xf = img.astype(np.float32).astype(np.float64)
    for d, s2 in ((1, 1.0), (3, 0.1), (5, 10.0)):
        c.launch("blur", grid, 128, X, Y, h, w, d, s2)
        c.sync()
        ref = oimg.blur(xf, d, s2)
        got = y.cpu().numpy().reshape(h, w).astype(np.float64)
        assert np.all(np.abs(got - ref) <= 1e-4 * np.abs(ref) + 1e-6), ("blur", d, float(np.abs(got - ref).max()))
    c.launch("sobel", grid, 128, X, Y, h, w)
    c.sync()
    ref = oimg.sobel(xf)
    got = y.cpu().numpy().reshape(h, w).astype(np.float64)
    assert np.all(np.abs(got - ref) <= 1e-4 * np.abs(ref) + 1e-5), ("sobel", float(np.abs(got - ref).max()))
    c.close()


# ------------------------------------------------------------------ conv1, edge shapes
@pytest.mark.parametrize("h,w,offset", [(1, 1, 0), (3, 5, 1), (33, 35, 0), (7, 4100, 0), (64, 130, 2),
                                        (517, 2051, 1), (2, 2048, 0), (9, 16386, 0)])
def test_conv1_edge_shapes(h, w, offset):
    """The product conv1 (two output rows per iteration, warp-transposed
    stores through shared memory, conv1.cuh) where warps run past the last
    column pair, W1 is odd (half-pixel stores masked), H1 is odd (the second
    row of the last pair absent), W % 4 != 0 / misaligned bases (scalar
    loads), and a CTA row block wider than one; against the fp64 oracle
    (R-DL: 3x3 stride 2 pad 1, ReLU), fp32 1e-4 relative + 1e-5 absolute."""
    c = D.Context(device=0)
    rng = np.random.default_rng(h * 131 + w)
    img = rng.random((h, w))
    wt = rng.uniform(-1, 1, size=72) / 3.0
    base = torch.zeros(h * w + 8, device="cuda")
    x = base[offset:offset + h * w]
    x.copy_(torch.from_numpy(img.astype(np.float32).ravel()))
    W1 = torch.from_numpy(wt.astype(np.float32)).cuda()
    h1, w1 = (h + 1) // 2, (w + 1) // 2
    y = torch.full((h1 * w1 * 8,), -7.0, device="cuda")
    torch.cuda.synchronize()
    X, Wt, Y = (c.register_tensor(k, t) for k, t in (("x", x), ("w", W1), ("y", y)))
    pairs = (w1 + 1) // 2
    grid = (max(1, -(-pairs // 256)), max(1, min((h1 + 1) // 2, 64)))
    c.launch("conv1", grid, 256, X, Wt, Y, h, w)
    c.sync()
    ref = odl.conv3x3s2(img.astype(np.float32).astype(np.float64),
                        wt.astype(np.float32).astype(np.float64).reshape(8, 3, 3, 1))
    got = y.cpu().numpy().reshape(h1, w1, 8).astype(np.float64)
    err = np.abs(got - ref) - (1e-4 * np.abs(ref) + 1e-5)
    assert np.all(err <= 0), float(err.max())
    c.close()


# ------------------------------------------------------------------ NORM, feature counts and ragged rows
@pytest.mark.parametrize("n,f", [(5923, 12), (1_000_003, 4), (777, 7), (40_000, 4), (3, 200), (20_011, 200)])
def test_norm_feature_counts(n, f):
    """The product NORM (cooperative; bulk-copy row ring when F % 4 == 0 and
    a block holds whole 2 RL-row chunks, the register path otherwise) for
    several F (ring slot sizes, G = F/4 column groups, the non-vector path
    at F = 7), ragged rows per block and ring tails; exact statistics and Z
    against the fp64 oracle (R-ML)."""
    from paper_2012_09646_b200.programs.img_ml import NORM_GRID, NORM_THREADS, norm_smem, norm_stats_bytes
    c = D.Context(device=0)
    rng = np.random.default_rng(n + f)
    X = rng.integers(-50, 50, size=(n, f), endpoint=True).astype(np.int32)
    tX = torch.from_numpy(X.ravel()).cuda()
    tZ = torch.zeros(n * f, device="cuda")
    st = torch.zeros(norm_stats_bytes(f), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    A, Z, S = (c.register_tensor(k, t) for k, t in (("X", tX), ("Z", tZ), ("s", st)))
    for _ in range(2):  # the grid barrier and exit counter reset for the next launch
        c.launch("norm", NORM_GRID, NORM_THREADS, A, Z, S, n, f, smem=norm_smem(f))
        c.sync()
    mu, sd = oml.norm_stats(X)
    stats = st[16:16 + 16 * f].view(torch.float64).cpu().numpy()
    assert np.allclose(stats[:f], mu, rtol=1e-12, atol=1e-12)
    assert np.allclose(1.0 / stats[f:], sd, rtol=1e-12)
    assert_close(tZ.cpu().numpy().reshape(n, f), oml.apply_norm(X, mu, sd), "Z")
    c.close()
