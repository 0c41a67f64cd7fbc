"""GPU parity (B200): IMG, ML, HITS, DL through the C ABI vs the fp64 oracle,
at small ragged sizes (several tiles + tails) and at BASELINE.json full size
(sampled outputs / properties), plus the synth GPU twin vs the host generator.

Criteria (north_star): DAG edges bit-exact;
integer labels bit-exact except oracle near-ties (top-2 gap <= 1e-5, which
must pick one of the tied classes); fp32 elementwise |g-o| <= 1e-4|o| +
1e-4 rms(o); fp32 reductions 1e-3 relative.
"""
import math

import numpy as np
import pytest
import torch

import synth
import synth.gpu as sg
from oracle import dl as odl
from oracle import hits as ohits
from oracle import img as oimg
from oracle import ml as oml
from paper_2012_09646_b200 import dagrt as D
from paper_2012_09646_b200.programs import DeepLearning, Hits, Images, MLEnsemble

pytestmark = pytest.mark.gpu


def close(g, o, rel=1e-4):
    o = np.asarray(o, np.float64)
    g = np.asarray(g, np.float64)
    rms = np.sqrt(np.mean(o * o)) if o.size else 0.0
    bad = np.abs(g - o) > rel * np.abs(o) + rel * rms
    return not bad.any(), (int(bad.sum()), float(np.max(np.abs(g - o))) if o.size else 0.0)


@pytest.fixture(scope="module")
def ctx():
    c = D.Context(device=0, record_dag=True)
    yield c
    c.close()


# ------------------------------------------------------------------ synth twin
@pytest.mark.parametrize("kind,args,dtype", [
    (synth.KIND_F32_UNIT, (), torch.float32),
    (synth.KIND_F64_RANGE, (30.0, 90.0), torch.float64),
    (synth.KIND_I32_BELOW, (10,), torch.int32),
    (synth.KIND_F32_SYM, (1.0 / math.sqrt(72.0),), torch.float32)])
def test_synth_gpu_twin_bit_exact(kind, args, dtype):
    n = 1_000_003
    t = torch.empty(n, dtype=dtype, device="cuda")
    spec = (kind, n, args)
    sg.fill_tensor(t, 77, "arr", spec)
    assert np.array_equal(t.cpu().numpy(), synth.draw(77, "arr", spec))


# ------------------------------------------------------------------ IMG
@pytest.mark.parametrize("h,w", [(1, 1), (7, 9), (65, 513), (200, 1100), (1024, 1024)])
def test_img_parity(ctx, h, w):
    p = Images(ctx, h=h, w=w)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    img = synth.draw(p.seed, "img", synth.spec_img(h, w)["img"]).reshape(h, w)
    o = oimg.img_pipeline(img)
    for name in ("bs", "bl", "bu", "ms", "iu", "i2", "i3"):
        ok, info = close(p.t[name].cpu().numpy().reshape(h, w), o[name])
        assert ok, (name, info)
    ok, info = close(p.t["ml"].cpu().numpy().reshape(h, w), o["ml"])
    assert ok, ("ml", info)
    mx = float(p.t["mx"][:4].view(torch.float32)[0])
    mn = float(p.t["mn"][:4].view(torch.float32)[0])
    assert abs(mx - o["mx"]) <= 1e-4 * abs(o["mx"]) + 1e-6
    assert abs(mn - o["mn"]) <= 1e-4 * abs(o["mx"]) + 1e-6


@pytest.mark.parametrize("prefetch", [True, False])
def test_img_stream_copy_precedes_all_readers(prefetch):
    """Stream mode: the input image (host-newer every run) is read by three
    blurs on three streams; its H2D must precede all of them, with and
    without the prefetcher.  The device copy is poisoned with NaN before the
    run, so a reader that is not ordered after the copy shows up as NaN."""
    from paper_2012_09646_b200 import dagrt as D
    c = D.Context(device=0, prefetch=prefetch)
    h = w = 2048
    p = Images(c, h=h, w=w, mode="stream")
    p.load_inputs(0)
    for _ in range(2):
        p.t["img"].fill_(float("nan"))
        torch.cuda.synchronize()
        p.run()
        c.sync()
        for name in ("bs", "bl", "bu", "i3"):
            assert not torch.isnan(p.t[name]).any(), name
    img = synth.draw(p.seed, "img", synth.spec_img(h, w)["img"]).reshape(h, w)
    o = oimg.img_pipeline(img)
    ok, info = close(p.t["i3"].cpu().numpy().reshape(h, w), o["i3"])
    assert ok, info
    del p
    c.close()
    torch.cuda.empty_cache()


def _img_chunk_oracle(seed, h, w, r0, r1):
    """Oracle over rows [r0, r1) of the full image (with a 4-row halo)."""
    a0, a1 = max(0, r0 - 4), min(h, r1 + 4)
    spec = synth.spec_img(h, w)["img"]
    idx = np.arange(a0 * w, a1 * w, dtype=np.uint64)
    img = synth.draw(seed, "img", spec, idx).reshape(a1 - a0, w).astype(np.float64)
    # zero padding only at the true image border: pad the halo-less sides
    bl = oimg.blur(img, *oimg.BLUR_L)
    ml = oimg.sobel(bl)
    lo, hi = r0 - a0, r1 - a0
    return img, ml[lo:hi], (a0, lo, hi)


def test_img_full_size_sampled(ctx):
    """16384^2 (BASELINE configs[2]), bench.py launch configuration: the global
    extrema over the full oracle sobel mask, and sampled rows of every stage."""
    h = w = 16384
    p = Images(ctx, h=h, w=w)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    mx_o, mn_o = -np.inf, np.inf
    sample_rows = [0, 1, 63, 64, 8191, 16320, 16383]
    checks = {}
    for r0 in range(0, h, 512):
        r1 = min(h, r0 + 512)
        img, ml, (a0, lo, hi) = _img_chunk_oracle(p.seed, h, w, r0, r1)
        mx_o = max(mx_o, float(ml.max()))
        mn_o = min(mn_o, float(ml.min()))
        for r in sample_rows:
            if r0 <= r < r1:
                checks[r] = (img, a0, r - a0)
    mx = float(p.t["mx"][:4].view(torch.float32)[0])
    mn = float(p.t["mn"][:4].view(torch.float32)[0])
    assert abs(mx - mx_o) <= 1e-4 * abs(mx_o)
    assert abs(mn - mn_o) <= 1e-4 * abs(mx_o)
    for r, (img, a0, k) in checks.items():
        bs = oimg.blur(img, *oimg.BLUR_S)
        bl = oimg.blur(img, *oimg.BLUR_L)
        bu = oimg.blur(img, *oimg.BLUR_U)
        ms = oimg.sobel(bs)
        ml = oimg.extend(oimg.sobel(bl), mx_o, mn_o)
        iu = oimg.unsharpen(img, bu)
        i3 = oimg.combine(oimg.combine(iu, bl, ml), bs, ms)
        for name, ref in (("bs", bs), ("bl", bl), ("ms", ms), ("ml", ml), ("i3", i3)):
            got = p.t[name][r * w:(r + 1) * w].cpu().numpy()
            ok, info = close(got, ref[k])
            assert ok, (name, r, info)
    del p
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ ML
def _ml_ref(p, X):
    pr = {k: v.astype(np.float64) for k, v in p.params.items()}
    return oml.ml(X, pr["theta"], pr["prior"], pr["W"], pr["b"])


def _check_labels(got, o):
    gap = oml.top2_gap(o["r1"], o["r2"])
    s = o["r1"] + o["r2"]
    tied = gap <= 1e-5
    exact = ~tied
    assert np.array_equal(got[exact], o["r"][exact])
    for i in np.nonzero(tied)[0]:
        assert s[i, got[i]] >= s[i].max() - 1e-5
    return int(tied.sum())


@pytest.mark.parametrize("n", [1, 37, 4099, 100_000])
def test_ml_parity(ctx, n):
    p = MLEnsemble(ctx, n=n)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    f, c = p.f, p.c
    X = synth.draw(p.seed, "X", synth.spec_ml_x(n, f)["X"]).reshape(n, f)
    o = _ml_ref(p, X)
    ok, info = close(p.t["Z"].cpu().numpy().reshape(n, f), o["Z"])
    assert ok, ("Z", info)
    ok, info = close(p.t["r1"].cpu().numpy().reshape(n, c), o["r1"])
    assert ok, ("r1", info)
    ok, info = close(p.t["r2"].cpu().numpy().reshape(n, c), o["r2"])
    assert ok, ("r2", info)
    ok, info = close(p.t["l"].cpu().numpy(), o["l"])
    assert ok, ("lse", info)
    _check_labels(p.t["r"].cpu().numpy(), o)


def test_ml_full_size_sampled(ctx):
    """10M x 200 (BASELINE configs[3]): exact oracle statistics over all of X
    (X is generator output, checked bit-equal to the host generator above),
    then the oracle on 20k sampled rows; NORM moments on all rows."""
    n, f = 10_000_000, 200
    p = MLEnsemble(ctx, n=n)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    X = p.t["X"].view(n, f).cpu().numpy()
    rng = np.random.default_rng(1)
    rows = np.sort(rng.choice(n, 20000, replace=False))
    rows[-1] = n - 1
    spec = synth.spec_ml_x(n, f)["X"]
    idx = (rows[:, None] * f + np.arange(f)[None, :]).ravel().astype(np.uint64)
    assert np.array_equal(X[rows], synth.draw(p.seed, "X", spec, idx).reshape(-1, f))
    mu, sd = oml.norm_stats(X)
    del X
    Xs = synth.draw(p.seed, "X", spec, idx).reshape(-1, f)
    pr = {k: v.astype(np.float64) for k, v in p.params.items()}
    Z = oml.apply_norm(Xs, mu, sd)
    r1 = oml.softmax(oml.exp_sub(*(lambda s: (s, oml.lse(s, oml.rowmax(s))))(
        oml.nb_mmul(Xs, pr["theta"], pr["prior"]))))
    r2 = oml.softmax(oml.addv(oml.mmul(Z, pr["W"]), pr["b"]))
    o = {"r1": r1, "r2": r2, "r": oml.argmax(r1, r2)}
    tr = torch.from_numpy(rows).cuda()
    ok, info = close(p.t["Z"].view(n, f)[tr].cpu().numpy(), Z)
    assert ok, ("Z", info)
    ok, info = close(p.t["r1"].view(n, 10)[tr].cpu().numpy(), r1)
    assert ok, ("r1", info)
    ok, info = close(p.t["r2"].view(n, 10)[tr].cpu().numpy(), r2)
    assert ok, ("r2", info)
    _check_labels(p.t["r"][tr].cpu().numpy(), o)
    Zd = p.t["Z"].view(n, f).double()
    assert torch.allclose(Zd.mean(0), torch.zeros(f, dtype=torch.float64, device="cuda"), atol=1e-5)
    assert torch.allclose(Zd.std(0, unbiased=False), torch.ones(f, dtype=torch.float64, device="cuda"),
                          atol=1e-5)
    del p, Zd
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ HITS
@pytest.mark.parametrize("n,e,seed", [(1, 5, 1), (5000, 15000, 2), (300_000, 900_000, 7)])
def test_powerlaw_graph_device_path_identical(n, e, seed):
    """The CUDA path of the graph generator (integer steps through torch)
    returns exactly the numpy path's CSR arrays."""
    a = synth.powerlaw_graph(seed, n, e)
    b = synth.powerlaw_graph(seed, n, e, device="auto")
    for x, y in zip(a, b):
        assert x.dtype == y.dtype and np.array_equal(x, y)


def _hits_check(p, graph, iters):
    ctx = p.ctx
    o = ohits.hits(*graph, iterations=iters)
    for name in ("a1", "h1"):
        ok, info = close(p.t[name].cpu().numpy(), o[name])
        assert ok, (name, info)
    an = float(p.t["an"][:4].view(torch.float32)[0])
    hn = float(p.t["hn"][:4].view(torch.float32)[0])
    assert abs(an - o["norms"][-1][0]) <= 1e-3 * o["norms"][-1][0] + 1e-30
    assert abs(hn - o["norms"][-1][1]) <= 1e-3 * o["norms"][-1][1] + 1e-30
    ok, info = close(p.vec("a2").cpu().numpy(), o["a2"])
    assert ok, ("a2", info)


@pytest.mark.parametrize("n,e", [(1, 0), (10, 30), (5000, 15000), (200_000, 600_000)])
def test_hits_parity(ctx, n, e):
    graph = synth.powerlaw_graph(5, n, e)
    p = Hits(ctx, n=n, e=e, iters=3, graph=graph)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    _hits_check(p, p.csr, 3)  # the registered (degree-ordered) graph


def test_hits_star_and_chain():
    """Hand-made graphs exercising rows spanning many SpMV tiles (a hub with
    20k out-edges) and empty rows."""
    c = D.Context(device=0)
    n = 30000
    src = np.concatenate([np.zeros(20000, np.int64), np.arange(1, 5000)])
    dst = np.concatenate([np.arange(1, 20001), np.arange(2, 5001)])
    import scipy.sparse as sp
    A = sp.csr_matrix((np.ones(len(src)), (src, dst)), shape=(n, n))
    A.sort_indices()
    At = A.T.tocsr()
    At.sort_indices()
    graph = (A.indptr.astype(np.int32), A.indices.astype(np.int32),
             At.indptr.astype(np.int32), At.indices.astype(np.int32))
    for order in ("degree", "given"):
        p = Hits(c, n=n, iters=2, graph=graph, vertex_order=order)
        p.load_inputs(0)
        p.run()
        c.sync()
        _hits_check(p, p.csr, 2)
        if order == "given":
            assert p.csr is graph and p.new_id is None
    c.close()


def test_hits_degree_order_is_a_relabelling():
    """The registered degree-ordered graph is P A P^T: the GPU scores in the
    registered order, mapped back through new_id, are the oracle's scores on
    the GIVEN graph (L882-886)."""
    n, e = 200_000, 600_000
    graph = synth.powerlaw_graph(9, n, e)
    c = D.Context(device=0)
    p = Hits(c, n=n, e=e, iters=3, graph=graph)
    assert p.new_id is not None and np.array_equal(np.sort(p.new_id), np.arange(n))
    p.load_inputs(0)
    p.run()
    c.sync()
    o = ohits.hits(*graph, iterations=3)
    for name in ("a1", "h1"):
        got = p.t[name].cpu().numpy()[p.new_id]  # back to the given ids
        ok, info = close(got, o[name])
        assert ok, (name, info)
    deg = np.diff(p.csr[0]) + np.diff(p.csr[2])
    assert np.all(np.diff(deg) <= 0)  # hubs first
    c.close()


def test_hits_full_size(ctx):
    """20M-vertex power-law graph (BASELINE configs[4]), 10 iterations, full
    oracle (every element)."""
    p = Hits(ctx)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    _hits_check(p, p.csr, p.iters)
    deg = np.diff(p.csr[0])
    assert deg.max() > 100_000  # the hub spans many merge-path tiles
    del p
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ DL
@pytest.mark.parametrize("h,w", [(1, 1), (9, 9), (19, 23), (64, 64), (515, 517), (1024, 1000)])
def test_dl_parity(ctx, h, w):
    p = DeepLearning(ctx, h=h, w=w)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    spec = synth.spec_dl(h, w)
    x = synth.draw(p.seed, "x", spec["x"]).reshape(h, w)
    y = synth.draw(p.seed, "y", spec["y"]).reshape(h, w)
    w1 = synth.draw(p.seed, "w1", spec["w1"])
    w2 = synth.draw(p.seed, "w2", spec["w2"])
    wd = synth.draw(p.seed, "wd", spec["wd"])
    o = odl.dl(x, y, w1, w2, wd)
    (h1, w1s), (h2, w2s), (h3, w3s) = p.shapes
    for name, shp in (("c1x", (h1, w1s, 8)), ("c1y", (h1, w1s, 8)), ("px", (h2, w2s, 8)),
                      ("c2x", (h3, w3s, 16)), ("c2y", (h3, w3s, 16))):
        if np.prod(shp) == 0:
            continue
        got = p.t[name][:int(np.prod(shp))].cpu().numpy().reshape(shp)
        ok, info = close(got, o[name])
        assert ok, (name, info)
    if o["z"].size:
        ok, info = close(p.t["z"][:o["z"].size].cpu().numpy(), o["z"])
        assert ok, ("z", info)
        assert abs(p.result() - o["r"]) <= 1e-3 * abs(o["r"]) + 1e-6


def test_dl_full_size_sampled(ctx):
    """2 x 16384^2 (BASELINE configs[4] DL): sampled conv2 outputs from the
    oracle on local input patches; r against the fp64 dot of the produced z."""
    h = w = 16384
    p = DeepLearning(ctx, h=h, w=w)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    spec = synth.spec_dl(h, w)
    w1 = synth.draw(p.seed, "w1", spec["w1"])
    w2 = synth.draw(p.seed, "w2", spec["w2"])
    (h1, w1s), (h2, w2s), (h3, w3s) = p.shapes
    rng = np.random.default_rng(3)
    pts = [(0, 0), (h3 - 1, w3s - 1), (0, w3s - 1)] + [tuple(rng.integers(0, h3, 2)) for _ in range(12)]
    for (pp, qq) in pts:
        # c2[pp,qq] needs p rows 2pp-1..2pp+1 -> c1 rows 4pp-2..4pp+3 -> x rows 8pp-5..8pp+7
        ylo, yhi = max(0, 8 * pp - 8), min(h, 8 * pp + 8)
        xlo, xhi = max(0, 8 * qq - 8), min(w, 8 * qq + 8)
        ys, xs = np.arange(ylo, yhi), np.arange(xlo, xhi)
        idx = (ys[:, None] * w + xs[None, :]).ravel().astype(np.uint64)
        xpatch = synth.draw(p.seed, "x", spec["x"], idx).reshape(len(ys), len(xs))
        # embed the patch at its true position parity so strides line up
        c1 = odl.conv3x3s2(np.pad(xpatch, ((ylo % 2, 0), (xlo % 2, 0))), w1.reshape(8, 3, 3, 1))
        # c1 local index a <-> global row (ylo - ylo%2)/2 + a
        g0r, g0c = (ylo - ylo % 2) // 2, (xlo - xlo % 2) // 2
        pool = odl.pool2x2(np.pad(c1, ((g0r % 2, 0), (g0c % 2, 0), (0, 0))))
        p0r, p0c = (g0r - g0r % 2) // 2, (g0c - g0c % 2) // 2
        # the needed pool entries lie >= 1 c1 row/col inside the patch, so the
        # patch's artificial zero border never reaches them
        acc = np.zeros(16)
        W2 = w2.reshape(16, 3, 3, 8).astype(np.float64)
        for a in range(3):
            for b in range(3):
                gy, gx = 2 * pp + a - 1, 2 * qq + b - 1
                if 0 <= gy < h2 and 0 <= gx < w2s:
                    acc += W2[:, a, b, :] @ pool[gy - p0r, gx - p0c, :]
        ref = np.maximum(acc, 0.0)
        got = p.t["c2x"][(pp * w3s + qq) * 16:(pp * w3s + qq + 1) * 16].cpu().numpy()
        ok, info = close(got, ref)
        assert ok, ((pp, qq), info, got, ref)
    z = p.t["z"].double()
    wd = p.t["wd"].double()
    r_ref = float((z * wd).sum())
    assert abs(p.result() - r_ref) <= 1e-3 * abs(r_ref)
    del p, z, wd
    torch.cuda.empty_cache()


@pytest.mark.parametrize("variant", ["conv2_ffma", "conv2_tc1", "conv2_tc2", "conv2_tc3", "conv2_tc4",
                                     "conv2_tc5", "conv2_tma0", "conv2_tma1", "conv2_tmag0", "conv2_tmag1",
                                     "conv2_tman1", "conv2_tmanr1", "conv2_tmar", "conv2_tman3x1"])
@pytest.mark.parametrize("h,w", [(19, 23), (515, 517)])
def test_dl_conv2_variants_match_oracle(ctx, exp, h, w, variant):
    """The other conv2 kernels (CUDA-core FFMA; the tcgen05 versions with a
    cp.async ring) against the oracle too."""
    p = DeepLearning(ctx, h=h, w=w)
    p.load_inputs(1)
    p.run()
    ctx.sync()
    (h1, w1s), (h2, w2s), (h3, w3s) = p.shapes
    out = torch.zeros(h3 * w3s * 16, device="cuda")
    torch.cuda.synchronize()
    o_arr = ctx.register_tensor(f"c2_{variant}_{h}", out)
    if variant == "conv2_ffma":
        ctx.launch(variant, ((w3s + 1) // 2 // 256 + 1, h3), 256, p.a["px"], p.a["w2"], o_arr, h2, w2s)
    elif variant in ("conv2_tc1", "conv2_tc3"):
        ctx.launch(variant, 2 * 148, 128, p.a["px"], p.a["w2"], o_arr, h2, w2s,
                   smem=2 * 9 * 512 + 2 * 9 * 4096 + 64)
    elif variant == "conv2_tman3x1":
        from paper_2012_09646_b200.programs.hits_dl import CONV2_TMAN_SMEM
        ctx.launch(variant, 148, 384, p.a["px"], p.a["w2"], o_arr, h2, w2s, smem=CONV2_TMAN_SMEM)
    elif variant == "conv2_tmar":
        from paper_2012_09646_b200.programs.hits_dl import CONV2_TMAR_SMEM, CONV2_TMAR_THREADS
        ctx.launch(variant, 148, CONV2_TMAR_THREADS, p.a["px"], p.a["w2"], o_arr, h2, w2s, smem=CONV2_TMAR_SMEM)
    elif variant.startswith("conv2_tmag") or variant.startswith("conv2_tman"):
        from paper_2012_09646_b200.programs.hits_dl import CONV2_TMAG_SMEM
        ctx.launch(variant, 148, 256, p.a["px"], p.a["w2"], o_arr, h2, w2s,
                   smem=CONV2_TMAG_SMEM[int(variant[-1])])
    elif variant.startswith("conv2_tma"):
        from paper_2012_09646_b200.programs.hits_dl import CONV2_TMA_SMEM
        ctx.launch(variant, 148, 128, p.a["px"], p.a["w2"], o_arr, h2, w2s,
                   smem=CONV2_TMA_SMEM[int(variant[-1])])
    elif variant == "conv2_tc2":
        ctx.launch(variant, 2 * 148, 256, p.a["px"], p.a["w2"], o_arr, h2, w2s,
                   smem=2 * 9 * 512 + 2 * 9 * 4096 + 64)
    elif variant == "conv2_tc4":
        ctx.launch(variant, 148, 128, p.a["px"], p.a["w2"], o_arr, h2, w2s,
                   smem=2 * 9 * 512 + 4 * 3 * 4 * 129 * 16 + 2 * 9 * 4096 + 64)
    else:
        from paper_2012_09646_b200.programs.hits_dl import CONV2_TC5_SMEM
        ctx.launch(variant, 148, 384, p.a["px"], p.a["w2"], o_arr, h2, w2s, smem=CONV2_TC5_SMEM)
    ctx.sync()
    spec = synth.spec_dl(h, w)
    w2 = synth.draw(p.seed, "w2", spec["w2"]).reshape(16, 3, 3, 8)
    px = p.t["px"][:h2 * w2s * 8].cpu().numpy().reshape(h2, w2s, 8)
    ref = odl.conv3x3s2(px, w2)
    ok, info = close(out.cpu().numpy().reshape(h3, w3s, 16), ref)
    assert ok, info
    ok, info = close(p.t["c2x"][:h3 * w3s * 16].cpu().numpy().reshape(h3, w3s, 16), ref)
    assert ok, info


@pytest.mark.parametrize("variant", ["conv1_b1", "conv1_b3", "conv1_b4", "conv1_b4cs", "conv1_r2b3cs",
                                     "conv1_r2b2"])
@pytest.mark.parametrize("h,w", [(19, 23), (515, 517)])
def test_dl_conv1_variants_bitwise(ctx, exp, h, w, variant):
    """Every conv1 variant (one or two output rows per iteration, store
    policies, register caps) gives the product kernel's output bit for bit
    (same arithmetic in the same order) -- the product is checked against the
    oracle in test_dl_parity."""
    p = DeepLearning(ctx, h=h, w=w)
    p.load_inputs(1)
    p.run()
    ctx.sync()
    (h1, w1s), _, _ = p.shapes
    out = torch.full_like(p.t["c1x"], -1.0)
    torch.cuda.synchronize()
    o_arr = ctx.register_tensor(f"c1_{variant}_{h}", out)
    L0 = p.L[0]
    rows = (h1 + 1) // 2 if "_r2" in variant else h1
    ctx.launch(variant, (L0.grid.x, max(1, min(rows, 7))), 256, p.a["x"], p.a["w1"], o_arr, h, w)
    ctx.sync()
    n = h1 * w1s * 8
    assert torch.equal(out[:n], p.t["c1x"][:n])


@pytest.mark.parametrize("h,w", [(515, 517)])
def test_tensor_core_truncates_fp32_to_tf32(ctx, exp, h, w):
    """Pins the hardware behaviour the product conv2 relies on: kind::tf32
    MMAs read an fp32 operand by TRUNCATING it to tf32.  conv2_tma1 (raw TMA
    box as A_hi, lo = x - trunc(x)) matches the oracle (test above) while
    conv2_tma2 (same kernel assuming round-to-nearest, lo = x - rn(x)) misses
    the tolerance on many outputs."""
    p = DeepLearning(ctx, h=h, w=w)
    p.load_inputs(1)
    p.run()
    ctx.sync()
    (h1, w1s), (h2, w2s), (h3, w3s) = p.shapes
    from paper_2012_09646_b200.programs.hits_dl import CONV2_TMA_SMEM
    out = torch.zeros(h3 * w3s * 16, device="cuda")
    torch.cuda.synchronize()
    o_arr = ctx.register_tensor(f"c2_rn_{h}", out)
    ctx.launch("conv2_tma2", 148, 128, p.a["px"], p.a["w2"], o_arr, h2, w2s, smem=CONV2_TMA_SMEM[2])
    ctx.sync()
    spec = synth.spec_dl(h, w)
    w2 = synth.draw(p.seed, "w2", spec["w2"]).reshape(16, 3, 3, 8)
    px = p.t["px"][:h2 * w2s * 8].cpu().numpy().reshape(h2, w2s, 8)
    ref = odl.conv3x3s2(px, w2)
    ok, info = close(out.cpu().numpy().reshape(h3, w3s, 16), ref)
    assert not ok, "round-to-nearest reading unexpectedly within tolerance"


@pytest.mark.parametrize("variant", ["spmv_sync", "spmv_as1", "spmv_x0s1", "spmv_x1s1"])
def test_spmv_merge_variants_bitwise(ctx, exp, variant):
    """The merge-path SpMV (previous default) and its variants (gathers in
    registers instead of cp.async; other L2 policies) give bit-identical y,
    and match the oracle."""
    from paper_2012_09646_b200.programs.hits_dl import spmv_out_bytes
    n, e = 300_000, 900_000
    rp, ci, _, _ = synth.powerlaw_graph(11, n, e)
    ob, grid = spmv_out_bytes(n, int(rp[-1]))
    t_rp = torch.from_numpy(rp).cuda()
    t_ci = torch.from_numpy(ci).cuda()
    t_x = torch.rand(n, device="cuda")
    y0 = torch.zeros(ob // 4 + 1, device="cuda")
    y1 = torch.zeros(ob // 4 + 1, device="cuda")
    torch.cuda.synchronize()
    A = [ctx.register_tensor(f"spv_{variant}_{k}", t) for k, t in
         (("rp", t_rp), ("ci", t_ci), ("x", t_x), ("y0", y0), ("y1", y1))]
    ctx.launch("spmv_merge", grid, 256, A[0], A[1], A[2], A[3], n)
    ctx.launch(variant, grid, 256, A[0], A[1], A[2], A[4], n)
    ctx.sync()
    assert torch.equal(y0[:n], y1[:n])
    ok, info = close(y0[:n].cpu().numpy(), ohits.spmv(rp, ci, t_x.cpu().numpy().astype(np.float64)))
    assert ok, info
    for a in A:
        ctx.unregister(a)


@pytest.mark.parametrize("n,e,seed", [(1, 0, 1), (1000, 0, 2), (5000, 200_000, 3), (300_000, 900_000, 11),
                                      (50_000, 2_000_000, 5)])
def test_spmv_plan_classes(ctx, exp, n, e, seed):
    """Row-class SpMV (alternative kernel) on graphs whose rows fall in every
    class (short, medium, long, multi-chunk hubs), run twice (the arrival
    counters must reset): matches the oracle and is bit-reproducible."""
    from paper_2012_09646_b200.programs.hits_dl import spmv_plan
    rp, ci, _, _ = synth.powerlaw_graph(seed, n, e) if e else (np.zeros(n + 1, np.int32),
                                                                np.zeros(0, np.int32), None, None)
    plan, grid, ws = spmv_plan(rp)
    t_rp = torch.from_numpy(rp).cuda()
    t_ci = torch.from_numpy(ci if ci.size else np.zeros(1, np.int32)).cuda()
    t_pl = torch.from_numpy(plan).cuda()
    t_x = torch.rand(n, device="cuda")
    y = torch.zeros((4 * n + ws) // 4 + 1, device="cuda")
    torch.cuda.synchronize()
    A = [ctx.register_tensor(f"spp_{n}_{e}_{k}", t) for k, t in
         (("rp", t_rp), ("ci", t_ci), ("pl", t_pl), ("x", t_x), ("y", y))]
    ctx.launch("spmv_plan", grid, 256, *A, n)
    ctx.sync()
    y1 = y[:n].clone()
    ctx.launch("spmv_plan", grid, 256, *A, n)
    ctx.sync()
    assert torch.equal(y1, y[:n])
    ok, info = close(y1.cpu().numpy(), ohits.spmv(rp, ci, t_x.cpu().numpy().astype(np.float64)))
    assert ok, info
    for a in A:
        ctx.unregister(a)
