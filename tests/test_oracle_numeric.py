"""Pins for the fp64 benchmark oracles (oracle/{vec,bs,img,ml,hits,dl}.py), no GPU.

Each test pins the oracle to something other than itself: a closed form, an
invariant, a special case that reduces to a library routine (scipy / numpy /
torch CPU fp64), or brute force -- chosen so that a dropped term, wrong sign,
wrong index or transposed operand fails at least one of them.
"""
import math

import numpy as np
import pytest
import scipy.ndimage as ndi
import scipy.sparse as sp
import scipy.special as ss

from oracle import bs as obs
from oracle import dl as odl
from oracle import hits as ohits
from oracle import img as oimg
from oracle import ml as oml
from oracle import vec as ovec

# ---------------------------------------------------------------- VEC


def test_vec_closed_form_harmonic():
    """x_i = 1/(i+1), y_i = 2/(i+1): z = -3 H_N^(2) = -3 (pi^2/6 - psi1(N+1))."""
    n = 1_000_000
    i = np.arange(n, dtype=np.float64)
    x, y = 1.0 / (i + 1), 2.0 / (i + 1)
    _, _, z = ovec.vec(x, y)
    exact = -3.0 * (math.pi ** 2 / 6.0 - ss.polygamma(1, n + 1))
    assert abs(z - exact) <= 1e-12 * abs(exact)
    assert abs(exact - (-4.934799200546)) < 1e-9  # SURVEY §8(c2) VEC printed value


def test_vec_squares_exact():
    x1, y1, z = ovec.vec([3.0, -2.0], [1.0, 0.5])
    assert list(x1) == [9.0, 4.0] and list(y1) == [1.0, 0.25]
    assert z == 9.0 + 4.0 - 1.0 - 0.25


# ---------------------------------------------------------------- B&S


def test_bs_cnd_within_as_bound():
    d = np.linspace(-8, 8, 200001)
    err = np.max(np.abs(obs.cnd(d) - ss.ndtr(d)))
    assert err <= 7.5e-8  # A&S 26.2.17 bound


def test_bs_call_matches_exact_black_scholes_within_bound():
    s = np.linspace(30, 90, 10001)
    sqt = math.sqrt(obs.T)
    d1 = (np.log(s / obs.K) + (obs.R + 0.5 * obs.V ** 2) * obs.T) / (obs.V * sqt)
    d2 = d1 - obs.V * sqt
    exact = s * ss.ndtr(d1) - obs.K * math.exp(-obs.R * obs.T) * ss.ndtr(d2)
    c = obs.call(s)
    assert np.all(np.abs(c - exact) <= (s + obs.K) * 7.5e-8)


def test_bs_put_call_parity():
    s = np.linspace(30, 90, 1001)
    c = obs.call(s)
    sqt = math.sqrt(obs.T)
    d1 = (np.log(s / obs.K) + (obs.R + 0.5 * obs.V ** 2) * obs.T) / (obs.V * sqt)
    d2 = d1 - obs.V * sqt
    put = obs.K * math.exp(-obs.R * obs.T) * obs.cnd(-d2) - s * obs.cnd(-d1)
    lhs = c - put
    rhs = s - obs.K * math.exp(-obs.R * obs.T)
    assert np.max(np.abs(lhs - rhs)) <= 2e-9 * 90


def test_bs_limits():
    kd = obs.K * math.exp(-obs.R * obs.T)
    assert abs(obs.call(np.array([1e6]))[0] - (1e6 - kd)) < 1e-6
    assert obs.call(np.array([1e-3]))[0] < 1e-12


# ---------------------------------------------------------------- IMG


def test_img_gaussian_closed_form():
    for d, s2 in (oimg.BLUR_S, oimg.BLUR_L, oimg.BLUR_U):
        g = oimg.gaussian(d, s2)
        r = d // 2
        assert abs(g.sum() - 1.0) < 1e-15
        assert abs(g[r, r + 1] / g[r, r] - math.exp(-1.0 / (2 * s2))) < 1e-14
        assert abs(g[r + 1, r + 1] / g[r, r] - math.exp(-2.0 / (2 * s2))) < 1e-14
        assert np.allclose(g, g.T) and np.allclose(g, g[::-1, ::-1])


def test_img_blur_and_sobel_equal_scipy_zero_padding():
    rng = np.random.default_rng(1)
    im = rng.random((7, 9))
    for d, s2 in (oimg.BLUR_S, oimg.BLUR_L, oimg.BLUR_U):
        ref = ndi.correlate(im, oimg.gaussian(d, s2), mode="constant", cval=0.0)
        assert np.allclose(oimg.blur(im, d, s2), ref, rtol=1e-13, atol=1e-14)
    gx = ndi.sobel(im, axis=1, mode="constant", cval=0.0)
    gy = ndi.sobel(im, axis=0, mode="constant", cval=0.0)
    assert np.allclose(oimg.sobel(im), np.hypot(gx, gy), rtol=1e-13, atol=1e-14)


def test_img_brute_force_7x9():
    rng = np.random.default_rng(2)
    im = rng.random((7, 9))
    g = oimg.gaussian(5, 10.0)
    out = np.zeros_like(im)
    for i in range(7):
        for j in range(9):
            acc = 0.0
            for a in range(-2, 3):
                for b in range(-2, 3):
                    if 0 <= i + a < 7 and 0 <= j + b < 9:
                        acc += g[a + 2, b + 2] * im[i + a, j + b]
            out[i, j] = acc
    assert np.allclose(oimg.blur(im, 5, 10.0), out, rtol=1e-13, atol=1e-15)


def test_img_constant_and_ramp():
    c = np.full((12, 12), 0.37)
    b = oimg.blur(c, 5, 10.0)
    assert np.allclose(b[2:-2, 2:-2], 0.37, atol=1e-15)
    assert np.allclose(oimg.sobel(c)[1:-1, 1:-1], 0.0, atol=1e-14)
    ramp = np.tile(np.arange(12, dtype=np.float64), (12, 1))  # I(i,j) = j
    assert np.allclose(oimg.sobel(ramp)[1:-1, 1:-1], 8.0, atol=1e-13)


def test_img_impulse_response_is_kernel():
    im = np.zeros((9, 9))
    im[4, 4] = 1.0
    assert np.allclose(oimg.blur(im, 5, 10.0)[2:7, 2:7], oimg.gaussian(5, 10.0), atol=1e-16)


def test_img_pointwise_special_cases():
    rng = np.random.default_rng(3)
    x, y = rng.random((5, 5)), rng.random((5, 5))
    assert np.array_equal(oimg.combine(x, y, np.ones((5, 5))), x)
    assert np.array_equal(oimg.combine(x, y, np.zeros((5, 5))), y)
    m = rng.random((5, 5))
    e = oimg.extend(m, m.max(), m.min())
    assert e.min() == 0.0 and e.max() <= 1.0
    assert np.all(e[m >= m.min() + (m.max() - m.min()) / 5.0] == 1.0)
    assert np.allclose(oimg.unsharpen(x, x), x)   # blur == image -> unchanged
    assert np.all(oimg.unsharpen(np.ones((2, 2)), np.zeros((2, 2))) == 1.0)  # clamp


# ---------------------------------------------------------------- ML


def _ml_inputs(n=257, f=oml.N_FEATURES, c=oml.N_CLASSES, seed=5):
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 10, size=(n, f)).astype(np.int32)
    theta = np.log(rng.dirichlet(np.ones(f), size=c))
    theta -= theta.mean(axis=0, keepdims=True)
    prior = np.full(c, math.log(1.0 / c))
    W = rng.uniform(-1, 1, size=(c, f)) / math.sqrt(f)
    b = rng.uniform(-1, 1, size=c)
    return X, theta, prior, W, b


def test_ml_mmul_equals_numpy_matmul():
    X, theta, prior, W, b = _ml_inputs()
    assert np.allclose(oml.mmul(X, theta), X.astype(np.float64) @ theta.T, rtol=1e-12, atol=1e-10)
    assert np.allclose(oml.nb_mmul(X, theta, prior), X @ theta.T + prior, rtol=1e-12, atol=1e-10)


def test_ml_norm_moments():
    X, *_ = _ml_inputs()
    Z = oml.norm(X)
    assert np.allclose(Z.mean(axis=0), 0.0, atol=1e-12)
    assert np.allclose(Z.std(axis=0), 1.0, atol=1e-12)
    Xc = X.copy()
    Xc[:, 3] = 4  # constant column -> zeros, no NaN
    assert np.all(oml.norm(Xc)[:, 3] == 0.0)


def test_ml_norm_stats_closed_forms_and_statistics_module():
    """NORM statistics pinned outside the oracle: an arithmetic progression
    0..n-1 has population variance (n^2 - 1)/12; a two-valued column {-a, a}
    in equal halves has mean 0 and sd a; wide-range columns (|x| up to 2^31)
    agree with Python's exact-rational statistics.pstdev."""
    import statistics
    n = 1001
    X = np.stack([np.arange(n), np.where(np.arange(n) % 2 == 0, -(1 << 30), 1 << 30)[:n],
                  np.full(n, 7)], axis=1).astype(np.int64)
    X[-1, 1] = 0  # odd n: make the two-valued column symmetric (mean 0)
    mu, sd = oml.norm_stats(X, chunk=97)
    assert mu[0] == (n - 1) / 2 and abs(sd[0] - math.sqrt((n * n - 1) / 12)) <= 1e-12 * sd[0]
    assert mu[1] == 0.0
    assert abs(sd[1] - math.sqrt(statistics.pvariance([int(v) for v in X[:, 1]]))) <= 1e-12 * sd[1]
    assert mu[2] == 7 and sd[2] == 1.0  # constant column: sd = 0 -> 1
    rng = np.random.default_rng(5)
    W = rng.integers(-(1 << 31), (1 << 31) - 1, size=(3000, 4), endpoint=True)
    mu, sd = oml.norm_stats(W.astype(np.int32), chunk=512)
    for j in range(4):
        col = [int(v) for v in W[:, j]]
        assert abs(mu[j] - statistics.fmean(col)) <= 1e-9 * (1 << 31) / 3000
        assert abs(sd[j] - statistics.pstdev(col)) <= 1e-12 * sd[j]


def test_ml_nb_posteriors_equal_scipy_softmax():
    X, theta, prior, W, b = _ml_inputs()
    out = oml.ml(X, theta, prior, W, b)
    ref = ss.softmax(X @ theta.T + prior, axis=1)
    assert np.allclose(out["r1_exp"], ref, rtol=1e-10, atol=1e-14)
    assert np.allclose(out["r1_exp"].sum(axis=1), 1.0, atol=1e-12)
    assert np.allclose(out["r1"], ss.softmax(ref, axis=1), rtol=1e-10)
    assert np.allclose(out["r2"], ss.softmax(oml.norm(X) @ W.T + b, axis=1), rtol=1e-10)
    assert np.allclose(out["r2"].sum(axis=1), 1.0, atol=1e-12)


def test_ml_argmax_brute_force_and_ties():
    X, theta, prior, W, b = _ml_inputs(n=64)
    out = oml.ml(X, theta, prior, W, b)
    s = out["r1"] + out["r2"]
    for i in range(64):
        best = 0
        for c in range(s.shape[1]):
            if s[i, c] > s[i, best]:
                best = c
        assert out["r"][i] == best
    r1 = np.array([[0.5, 0.5, 0.0]])
    r2 = np.array([[0.0, 0.0, 0.0]])
    assert oml.argmax(r1, r2)[0] == 0


# ---------------------------------------------------------------- HITS


def _csr(n, edges):
    A = sp.csr_matrix((np.ones(len(edges)), ([e[0] for e in edges], [e[1] for e in edges])),
                      shape=(n, n))
    A.sort_indices()
    At = A.T.tocsr()
    At.sort_indices()
    return A, (A.indptr, A.indices, At.indptr, At.indices)


def test_hits_spmv_equals_scipy():
    rng = np.random.default_rng(9)
    n = 50
    edges = {(int(a), int(b)) for a, b in rng.integers(0, n, size=(300, 2)) if a != b}
    A, (rp, ci, rpt, cit) = _csr(n, sorted(edges))
    x = rng.random(n)
    assert np.allclose(ohits.spmv(rp, ci, x), A @ x, rtol=1e-14)
    assert np.allclose(ohits.spmv(rpt, cit, x), A.T @ x, rtol=1e-14)


def test_hits_converges_to_principal_eigenvectors():
    rng = np.random.default_rng(11)
    n = 30
    edges = {(int(a), int(b)) for a, b in rng.integers(0, n, size=(120, 2)) if a != b}
    A, csr = _csr(n, sorted(edges))
    Ad = A.toarray()
    ev, V = np.linalg.eigh(Ad.T @ Ad)
    gap = ev[-2] / ev[-1]
    assert gap < 0.8
    out = ohits.hits(*csr, iterations=200)
    a = out["a1"]
    va = np.abs(V[:, -1])
    assert abs(np.linalg.norm(a) - 1.0) < 1e-12 and abs(np.linalg.norm(out["h1"]) - 1.0) < 1e-12
    assert np.allclose(a, va, atol=1e-8)
    evh, Vh = np.linalg.eigh(Ad @ Ad.T)
    assert np.allclose(out["h1"], np.abs(Vh[:, -1]), atol=1e-8)
    for an, hn in out["norms"][1:]:
        assert an > 0 and hn > 0


def test_hits_cycle_and_bipartite():
    n = 7
    _, csr = _csr(n, [(i, (i + 1) % n) for i in range(n)])
    out = ohits.hits(*csr, iterations=3)
    assert np.allclose(out["a1"], 1 / math.sqrt(n)) and np.allclose(out["h1"], 1 / math.sqrt(n))
    m, k = 3, 4
    edges = [(i, m + j) for i in range(m) for j in range(k)]
    _, csr = _csr(m + k, edges)
    out = ohits.hits(*csr, iterations=4)
    assert np.allclose(out["a1"][m:], 1 / math.sqrt(k)) and np.allclose(out["a1"][:m], 0)
    assert np.allclose(out["h1"][:m], 1 / math.sqrt(m)) and np.allclose(out["h1"][m:], 0)


def test_hits_empty_graph_zero_norm():
    n = 4
    rp = np.zeros(n + 1, dtype=np.int32)
    ci = np.zeros(0, dtype=np.int32)
    out = ohits.hits(rp, ci, rp, ci, iterations=2)
    assert np.all(out["a1"] == 0) and np.all(out["h1"] == 0)


# ---------------------------------------------------------------- DL


def test_dl_conv_equals_torch_conv2d_fp64():
    import torch
    rng = np.random.default_rng(13)
    for (h, w) in ((9, 9), (10, 7), (16, 16)):
        x = rng.random((h, w, 8))
        wt = rng.uniform(-1, 1, size=(16, 3, 3, 8))
        ref = torch.nn.functional.conv2d(torch.from_numpy(x).permute(2, 0, 1)[None],
                                         torch.from_numpy(wt).permute(0, 3, 1, 2),
                                         stride=2, padding=1)
        ref = torch.relu(ref)[0].permute(1, 2, 0).numpy()
        assert np.allclose(odl.conv3x3s2(x, wt), ref, rtol=1e-12, atol=1e-13)


def test_dl_delta_kernel_and_pool():
    rng = np.random.default_rng(14)
    x = rng.random((9, 9))
    w = np.zeros((8, 3, 3, 1))
    w[:, 1, 1, 0] = 1.0  # delta at the centre tap
    out = odl.conv3x3s2(x, w)
    for k in range(8):
        assert np.array_equal(out[:, :, k], x[0::2, 0::2])
    c = np.full((6, 8, 3), 0.7)
    assert np.allclose(odl.pool2x2(c), 0.7)
    t = np.arange(16.0).reshape(4, 4, 1)
    assert odl.pool2x2(t)[0, 0, 0] == (0 + 1 + 4 + 5) / 4.0


def test_dl_dot_and_concat():
    rng = np.random.default_rng(15)
    a, b = rng.random((3, 4, 16)), rng.random((3, 4, 16))
    z = odl.concat(a, b)
    assert z[0] == a[0, 0, 0] and z[16] == a[0, 1, 0] and z[a.size] == b[0, 0, 0]
    wd = rng.uniform(-1, 1, z.size)
    assert abs(odl.dot(z, wd) - math.fsum(z * wd)) < 1e-12


@pytest.mark.parametrize("h", [9, 12])
def test_dl_pipeline_shapes(h):
    rng = np.random.default_rng(16)
    x, y = rng.random((h, h)), rng.random((h, h))
    w1 = rng.uniform(-1, 1, 72)
    w2 = rng.uniform(-1, 1, 16 * 72)
    h1 = (h + 1) // 2
    h3 = (h1 // 2 + 1) // 2
    wd = rng.uniform(-1, 1, 2 * h3 * h3 * 16)
    out = odl.dl(x, y, w1, w2, wd)
    assert out["c1x"].shape == (h1, h1, 8) and out["c2x"].shape == (h3, h3, 16)
    assert np.all(out["c1x"] >= 0)
