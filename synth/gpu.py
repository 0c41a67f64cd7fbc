"""GPU fills with the shared generator (libsynth.so, synth/csrc/synth.cu)."""
import ctypes as C
import os

import synth

_L = None


def lib():
    global _L
    if _L is None:
        p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
        if not os.path.exists(p):
            raise ImportError(f"{p} not built: run `python -m paper_2012_09646_b200.build`")
        _L = C.CDLL(p)
        _L.synth_fill.argtypes = [C.c_void_p, C.c_longlong, C.c_int, C.c_ulonglong, C.c_double,
                                  C.c_double, C.c_longlong, C.c_void_p]
        _L.synth_fill.restype = C.c_int
        _L.synth_sync.restype = C.c_int
    return _L


def fill(dev_ptr, seed, name, spec, idx0=0, n=None, sync=True):
    """Fill device memory with elements [idx0, idx0+n) of array ``name``."""
    kind, total, args = spec
    n = total if n is None else n
    a = list(args) + [0.0, 0.0]
    if kind == synth.KIND_F64_RANGE:
        a0, a1 = float(args[0]), float(args[1])
    else:
        a0, a1 = float(a[0]), float(a[1])
    r = lib().synth_fill(C.c_void_p(dev_ptr), n, kind, synth.key(seed, name), a0, a1, idx0, None)
    if r:
        raise RuntimeError(f"synth_fill failed: cuda error {r}")
    if sync:
        r = lib().synth_sync()
        if r:
            raise RuntimeError(f"synth_sync failed: cuda error {r}")


def fill_tensor(t, seed, name, spec):
    """Fill the first spec[1] elements of t (allocations may be padded to >= 1)."""
    assert t.numel() >= spec[1], (t.numel(), spec[1])
    if spec[1]:
        fill(t.data_ptr(), seed, name, spec)
