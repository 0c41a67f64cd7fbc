"""Whole-program parity against the fp64 oracle (test helper, GPU side).

``check(p, set_index)`` compares every output of a benchmark program that
has just run (any policy: parallel, serial-sync, single-stream children,
graph cache, hand-written CUDA graph) with the oracle on the same seeded
inputs.  Criteria are the north_star's:
fp32 elementwise |g-o| <= 1e-4|o| + 1e-4 rms(o); fp32 reductions 1e-3
relative; fp64 (B&S) 1e-10 relative + 1e-12 absolute; integer labels
bit-exact except oracle near-ties (top-2 gap <= 1e-5).
"""
import numpy as np
import torch

import synth
from oracle import bs as obs
from oracle import dl as odl
from oracle import hits as ohits
from oracle import img as oimg
from oracle import ml as oml
from oracle import vec as ovec


def close(g, o, rel=1e-4):
    o = np.asarray(o, np.float64)
    g = np.asarray(g, np.float64)
    rms = np.sqrt(np.mean(o * o)) if o.size else 0.0
    bad = ~(np.abs(g - o) <= rel * np.abs(o) + rel * rms)
    return not bad.any(), (int(bad.sum()), float(np.nanmax(np.abs(g - o))) if o.size else 0.0)


def assert_close(g, o, what, rel=1e-4):
    ok, info = close(g, o, rel)
    assert ok, (what, info)


def red(t):
    """fp32 result of a scalar-reduction output array (RedOut)."""
    return float(t[:4].view(torch.float32)[0])


def check_labels(got, o):
    gap = oml.top2_gap(o["r1"], o["r2"])
    s = o["r1"] + o["r2"]
    tied = gap <= 1e-5
    assert np.array_equal(got[~tied], o["r"][~tied])
    for i in np.nonzero(tied)[0]:
        assert s[i, got[i]] >= s[i].max() - 1e-5
    return int(tied.sum())


def check_vec(p, seed):
    spec = synth.spec_vec(p.n)
    x1, y1, z = ovec.vec(synth.draw(seed, "x", spec["x"]), synth.draw(seed, "y", spec["y"]))
    assert_close(p.t["x1"].cpu().numpy(), x1, "x1")
    assert_close(p.t["y1"].cpu().numpy(), y1, "y1")
    assert abs(red(p.t["z"]) - z) <= 1e-3 * abs(z) + 1e-30, (red(p.t["z"]), z)


def check_bs(p, seed):
    sp = synth.spec_bs(p.n, p.nvec)
    for i in range(p.nvec):
        s = synth.draw(seed, f"s{i}", sp[f"s{i}"])
        out = p.t[f"c{i}"].cpu().numpy()
        if getattr(p, "dtype", "f64") == "f32":  # fp32 variant: the fp32 criterion on the rounded prices
            assert_close(out, obs.call(s.astype(np.float32).astype(np.float64)), ("bs_f32", i))
            continue
        ref = obs.call(s)
        err = np.abs(out - ref) - (1e-10 * np.abs(ref) + 1e-12)
        assert np.all(err <= 0), (i, float(err.max()))


def check_img(p, seed):
    h, w = p.h, p.w
    img = synth.draw(seed, "img", synth.spec_img(h, w)["img"]).reshape(h, w)
    o = oimg.img_pipeline(img)
    for name in ("bs", "bl", "bu", "ms", "ml", "iu", "i2", "i3"):
        assert_close(p.t[name].cpu().numpy().reshape(h, w), o[name], name)
    assert abs(red(p.t["mx"]) - o["mx"]) <= 1e-4 * abs(o["mx"]) + 1e-6
    assert abs(red(p.t["mn"]) - o["mn"]) <= 1e-4 * abs(o["mx"]) + 1e-6


def check_ml(p, seed, X=None):
    n, f, c = p.n, p.f, p.c
    if X is None:
        X = synth.draw(seed, "X", synth.spec_ml_x(n, f)["X"]).reshape(n, f)
    pr = {k: v.astype(np.float64) for k, v in p.params.items()}
    o = oml.ml(X, pr["theta"], pr["prior"], pr["W"], pr["b"])
    assert_close(p.t["Z"].cpu().numpy().reshape(n, f), o["Z"], "Z")
    assert_close(p.t["r1"].cpu().numpy().reshape(n, c), o["r1"], "r1")
    assert_close(p.t["r2"].cpu().numpy().reshape(n, c), o["r2"], "r2")
    assert_close(p.t["l"].cpu().numpy(), o["l"], "lse")
    return check_labels(p.t["r"].cpu().numpy(), o)


def check_hits(p, seed=None):
    o = ohits.hits(*p.csr, iterations=p.iters)
    for name in ("a1", "h1"):
        assert_close(p.t[name].cpu().numpy(), o[name], name)
    an, hn = red(p.t["an"]), red(p.t["hn"])
    assert abs(an - o["norms"][-1][0]) <= 1e-3 * o["norms"][-1][0] + 1e-30
    assert abs(hn - o["norms"][-1][1]) <= 1e-3 * o["norms"][-1][1] + 1e-30
    assert_close(p.vec("a2").cpu().numpy(), o["a2"], "a2")


def dl_oracle(p, seed):
    h, w = p.h, p.w
    spec = synth.spec_dl(h, w)
    x = synth.draw(seed, "x", spec["x"]).reshape(h, w)
    y = synth.draw(seed, "y", spec["y"]).reshape(h, w)
    base = p.seed  # weights are drawn from set 0
    w1 = synth.draw(base, "w1", spec["w1"])
    w2 = synth.draw(base, "w2", spec["w2"])
    wd = synth.draw(base, "wd", spec["wd"])
    return odl.dl(x, y, w1, w2, wd)


def check_dl(p, seed):
    o = dl_oracle(p, seed)
    (h1, w1s), (h2, w2s), (h3, w3s) = p.shapes
    for name, shp in (("c1x", (h1, w1s, 8)), ("c1y", (h1, w1s, 8)), ("px", (h2, w2s, 8)),
                      ("py", (h2, w2s, 8)), ("c2x", (h3, w3s, 16)), ("c2y", (h3, w3s, 16))):
        if np.prod(shp) == 0:
            continue
        got = p.t[name][:int(np.prod(shp))].cpu().numpy().reshape(shp)
        assert_close(got, o[name], name)
    if o["z"].size:
        assert_close(p.t["z"][:o["z"].size].cpu().numpy(), o["z"], "z")
        assert abs(red(p.t["r"]) - o["r"]) <= 1e-3 * abs(o["r"]) + 1e-6, (red(p.t["r"]), o["r"])
    return o


CHECKS = {"vec": check_vec, "bs": check_bs, "img": check_img, "ml": check_ml, "hits": check_hits,
          "dl": check_dl}


def check(p, set_index=0):
    """Oracle parity of every output of program ``p`` run on input set ``set_index``."""
    return CHECKS[p.name](p, p.seed + set_index)
