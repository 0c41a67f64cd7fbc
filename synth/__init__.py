"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module is the ONE piece of code both sides may use (task rule ③): it
generates the benchmark inputs and holds none of the method's arithmetic --
no DAG logic, no kernel math.  Every value is a pure function of
(seed, array name, element index) through a counter-based generator, so

* the oracle can draw any element (or a sample of elements) on the host with
  numpy, and
* the GPU side can draw the same full-size arrays in HBM with
  ``synth/csrc/synth.cu`` (libsynth.so), which implements the identical
  generator bit for bit (checked by ``tests/test_synth.py`` on the GPU).

Generator: the SplitMix64 output function applied to ``key + (i+1)*GOLDEN``
(mod 2**64), with ``key = mix(seed*GOLDEN ^ fnv1a64(name))``.

Input recipes follow SURVEY.md §8(d): the paper
only says "random data" and gives the shapes per
benchmark (L860-891, Table I).
"""
from __future__ import annotations

import math

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1
BASE_SEED = 20120964  # seed = 20120964 + set_index

_G = np.uint64(GOLDEN)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def fnv1a64(name: str) -> int:
    h = 0xCBF29CE484222325
    for b in name.encode():
        h ^= b
        h = (h * 0x100000001B3) & M64
    return h


def _fin_int(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def key(seed: int, name: str) -> int:
    """64-bit stream key of array ``name`` under ``seed``."""
    return _fin_int(((seed * GOLDEN) & M64) ^ fnv1a64(name))


def bits(k: int, idx) -> np.ndarray:
    """Raw 64-bit draws for element indices ``idx`` (uint64 array)."""
    i = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(k) + (i + np.uint64(1)) * _G
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


# --- distributions (all exact integer / single-rounding recipes, mirrored in synth.cu)

def f32_unit(k, idx):
    """U[0,1) float32: top 24 bits * 2^-24 (exact)."""
    return ((bits(k, idx) >> np.uint64(40)).astype(np.float64) * 2.0**-24).astype(np.float32)


def f64_unit(k, idx):
    """U[0,1) float64: top 53 bits * 2^-53 (exact)."""
    return (bits(k, idx) >> np.uint64(11)).astype(np.float64) * 2.0**-53


def f64_range(k, idx, lo: float, hi: float):
    """U[lo,hi) float64 = lo + (hi-lo)*u, two IEEE roundings (no FMA)."""
    return np.float64(lo) + np.float64(hi - lo) * f64_unit(k, idx)


def f32_sym(k, idx, scale: float):
    """float32((2u-1)*scale) with u = f64_unit: symmetric U(-scale, scale)."""
    u = f64_unit(k, idx)
    return ((2.0 * u - 1.0) * np.float64(scale)).astype(np.float32)


def i32_below(k, idx, m: int):
    """Integer U{0..m-1}: ((h>>32)*m)>>32 (exact)."""
    h = bits(k, idx) >> np.uint64(32)
    with np.errstate(over="ignore"):
        return ((h * np.uint64(m)) >> np.uint64(32)).astype(np.int32)


def _full(n):
    return np.arange(n, dtype=np.uint64)


# ------------------------------------------------------------------ recipes
# Each recipe returns host numpy arrays in the GPU storage dtype.  Names are
# the array names of the benchmark programs; the GPU fills use the same
# (seed, name) keys through libsynth.so.

# Generator "kinds" understood by synth.cu (same numbering there).
KIND_F32_UNIT, KIND_F64_RANGE, KIND_I32_BELOW, KIND_F32_SYM = 0, 1, 2, 3


def spec_vec(n: int):
    """VEC: x, y ~ U[0,1) fp32, length n."""
    return {"x": (KIND_F32_UNIT, n, ()), "y": (KIND_F32_UNIT, n, ())}


BS_NVEC = 10  # "10 underlying stocks, and 10 vectors of prices"


def spec_bs(n: int, nvec: int = BS_NVEC):
    """B&S (L865-870): S_i ~ U[30,90) fp64 per option (SURVEY §8(c) prop.)."""
    return {f"s{i}": (KIND_F64_RANGE, n, (30.0, 90.0)) for i in range(nvec)}


def spec_img(h: int, w: int):
    """IMG (L871-875): one row-major fp32 image ~ U[0,1)."""
    return {"img": (KIND_F32_UNIT, h * w, ())}


def spec_dl(h: int, w: int):
    """DL (L887-891): two fp32 images ~ U[0,1) + weights ~ U(-1,1)/sqrt(fan_in)."""
    h1, w1 = (h + 1) // 2, (w + 1) // 2       # conv1 3x3 s2 p1
    h2, w2 = h1 // 2, w1 // 2                 # mean-pool 2x2 s2
    h3, w3 = (h2 + 1) // 2, (w2 + 1) // 2     # conv2 3x3 s2 p1
    nz = 2 * h3 * w3 * 16
    return {
        "x": (KIND_F32_UNIT, h * w, ()),
        "y": (KIND_F32_UNIT, h * w, ()),
        "w1": (KIND_F32_SYM, 8 * 9 * 1, (1.0 / math.sqrt(9.0),)),
        "w2": (KIND_F32_SYM, 16 * 9 * 8, (1.0 / math.sqrt(72.0),)),
        "wd": (KIND_F32_SYM, nz, (1.0 / math.sqrt(float(max(nz, 1))),)),
    }


def spec_ml_x(n: int, f: int):
    """ML (L876-881): X ~ U{0..9} int32, n rows x f features (row-major)."""
    return {"X": (KIND_I32_BELOW, n * f, (10,))}


def draw(seed: int, name: str, spec, idx=None):
    """Draw array ``name`` of ``spec`` (optionally only elements ``idx``)."""
    kind, n, args = spec
    k = key(seed, name)
    ii = _full(n) if idx is None else np.asarray(idx, dtype=np.uint64)
    if kind == KIND_F32_UNIT:
        return f32_unit(k, ii)
    if kind == KIND_F64_RANGE:
        return f64_range(k, ii, *args)
    if kind == KIND_I32_BELOW:
        return i32_below(k, ii, *args)
    if kind == KIND_F32_SYM:
        return f32_sym(k, ii, *args)
    raise ValueError(kind)


def ml_params(seed: int, f: int, c: int):
    """Synthetic trained ML parameters (small; always host-generated).

    NB: theta[c,:] = log(u_c / sum u_c), u ~ U(0,1], then centred per feature
    across classes (SURVEY §8(c) "Numerical conditioning": posteriors are
    unchanged in exact arithmetic).  prior = log(1/C).
    RR: W ~ U(-1,1)/sqrt(F), b ~ U(-1,1).
    Returned as float32 (GPU storage dtype).
    """
    u = (f64_unit(key(seed, "theta"), _full(c * f)).reshape(c, f) + 2.0**-54)
    theta = np.log(u / u.sum(axis=1, keepdims=True))
    theta = theta - theta.mean(axis=0, keepdims=True)
    prior = np.full(c, math.log(1.0 / c))
    w = f32_sym(key(seed, "W"), _full(c * f), 1.0 / math.sqrt(f)).reshape(c, f)
    b = f32_sym(key(seed, "b"), _full(c), 1.0)
    return {"theta": theta.astype(np.float32), "prior": prior.astype(np.float32),
            "W": w, "b": b}


def powerlaw_graph(seed: int, n: int, e_target: int, alpha: float = 2.1, device=None):
    """Chung-Lu style power-law digraph (SURVEY §8(d) HITS recipe).

    Sources and destinations drawn i.i.d. with P(i) ~ (i+1)^(-1/(alpha-1)),
    relabelled by a seeded permutation; duplicates and self loops removed.
    Returns (row_ptr, col_idx) of A and (row_ptr_t, col_idx_t) of A^T, int32,
    with column indices sorted within each row.

    ``device``: None = numpy on the host; "auto" = a CUDA device through torch
    when one is present (the full 20M-vertex graph takes minutes in numpy).
    Both paths use only exact integer operations after the identical fp64
    draws and cdf (searchsorted, stable sort on the unsigned keys, unique,
    sort), so they return the same arrays (tests/test_synth.py).
    """
    expo = -1.0 / (alpha - 1.0)
    w = np.power(np.arange(1, n + 1, dtype=np.float64), expo)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    us = f64_unit(key(seed, "src"), _full(e_target))
    ud = f64_unit(key(seed, "dst"), _full(e_target))
    pkeys = bits(key(seed, "perm"), _full(n))
    if device == "auto":
        try:
            import torch
            if torch.cuda.is_available():
                return _powerlaw_torch(cdf, us, ud, pkeys, n)
        except ImportError:
            pass
    src = np.minimum(np.searchsorted(cdf, us, side="right"), n - 1).astype(np.int64)
    dst = np.minimum(np.searchsorted(cdf, ud, side="right"), n - 1).astype(np.int64)
    del us, ud
    # seeded permutation: argsort of random keys
    perm = np.argsort(pkeys, kind="stable").astype(np.int64)
    src = perm[src]
    dst = perm[dst]
    keep = src != dst
    code = np.unique(src[keep] * n + dst[keep])
    del src, dst, keep
    r = (code // n).astype(np.int64)
    c = (code % n).astype(np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=row_ptr[1:])
    # transpose: sort by (c, r)
    order = np.lexsort((r, c))
    rt = c[order].astype(np.int64)
    ct = r[order].astype(np.int32)
    row_ptr_t = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rt, minlength=n), out=row_ptr_t[1:])
    assert row_ptr[-1] < 2**31
    return (row_ptr.astype(np.int32), c, row_ptr_t.astype(np.int32), ct)


def _powerlaw_torch(cdf, us, ud, pkeys, n):
    """The integer steps of powerlaw_graph on a CUDA device (same results)."""
    import torch
    dev = torch.device("cuda")
    tc = torch.from_numpy(cdf).to(dev)
    src = torch.clamp(torch.searchsorted(tc, torch.from_numpy(us).to(dev), right=True), max=n - 1)
    dst = torch.clamp(torch.searchsorted(tc, torch.from_numpy(ud).to(dev), right=True), max=n - 1)
    del tc
    # unsigned order of the 64-bit keys = signed order with the sign bit flipped
    sk = torch.from_numpy((pkeys ^ np.uint64(1 << 63)).view(np.int64)).to(dev)
    perm = torch.sort(sk, stable=True).indices
    del sk
    src = perm[src]
    dst = perm[dst]
    keep = src != dst
    code = torch.unique(src[keep] * n + dst[keep], sorted=True)
    del src, dst, keep, perm
    r = code // n
    c = code % n
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    row_ptr[1:] = torch.cumsum(torch.bincount(r, minlength=n), 0)
    # transpose: (c, r) order = sort of c*n + r (unique codes)
    codet = torch.sort(c * n + r).values
    rt = codet // n
    ct = codet % n
    row_ptr_t = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    row_ptr_t[1:] = torch.cumsum(torch.bincount(rt, minlength=n), 0)
    assert int(row_ptr[-1]) < 2**31
    out = tuple(t.to(torch.int32).cpu().numpy() for t in (row_ptr, c, row_ptr_t, ct))
    torch.cuda.synchronize()
    return out
