"""The shared seeded input generator (synth/), host side, no GPU.

The numpy vectorised generator is checked against a scalar pure-Python
SplitMix64 (the published constants), so the CUDA twin in synth/csrc can be
checked against either.
"""
import numpy as np

import synth

M = (1 << 64) - 1


def _scalar(k, i):
    z = (k + (i + 1) * 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_bits_match_scalar_splitmix():
    k = synth.key(synth.BASE_SEED, "x")
    idx = [0, 1, 2, 1000, 2**40 + 3]
    got = synth.bits(k, idx)
    assert [int(v) for v in got] == [_scalar(k, i) for i in idx]
    # SplitMix64 seeded with 0: first output 0xE220A8397B1DCDAF (published reference)
    assert int(synth.bits(0, [0])[0]) == 0xE220A8397B1DCDAF


def test_distributions_ranges():
    k = synth.key(1, "a")
    idx = np.arange(100000)
    u = synth.f32_unit(k, idx)
    assert u.dtype == np.float32 and u.min() >= 0 and u.max() < 1
    r = synth.f64_range(k, idx, 30.0, 90.0)
    assert r.min() >= 30 and r.max() < 90 and abs(r.mean() - 60) < 0.5
    i = synth.i32_below(k, idx, 10)
    assert i.min() == 0 and i.max() == 9 and np.all(np.bincount(i) > 9000)
    s = synth.f32_sym(k, idx, 0.5)
    assert s.min() >= -0.5 and s.max() <= 0.5


def test_draw_subset_equals_full():
    spec = synth.spec_bs(1000)["s3"]
    full = synth.draw(7, "s3", spec)
    idx = np.array([0, 5, 999])
    assert np.array_equal(synth.draw(7, "s3", spec, idx), full[idx])


def test_powerlaw_graph_csr_valid():
    rp, ci, rpt, cit = synth.powerlaw_graph(3, 2000, 6000)
    n = 2000
    assert rp[0] == 0 and rp[-1] == len(ci) and len(rp) == n + 1
    assert rpt[-1] == len(cit) == len(ci)
    assert np.all(np.diff(rp) >= 0)
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.all(rows != ci)  # no self loops
    code = rows.astype(np.int64) * n + ci
    assert len(np.unique(code)) == len(code)  # no duplicates
    rows_t = np.repeat(np.arange(n), np.diff(rpt))
    code_t = cit.astype(np.int64) * n + rows_t
    assert np.array_equal(np.sort(code), np.sort(code_t))  # A^T is the transpose
    deg = np.diff(rp) + np.diff(rpt)
    assert deg.max() > 20 * deg.mean()  # heavy tail
