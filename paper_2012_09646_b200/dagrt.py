"""Thin ctypes binding of libdagrt.so (include/dagrt.h) -- argument
marshalling only.  Every step of the hot path (dependency inference, stream
assignment, event wiring, transfers, kernels) runs in the native library.

PyTorch is used by callers only for device memory, pinned host memory and
streams; this module never falls back to any Python or CPU computation: if
the native library is missing it raises.
"""
from __future__ import annotations

import ctypes as C
import functools
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.path.join(HERE, "libdagrt.so")

OK, EINVAL, ENOTFOUND, EALIAS, ESIG, ESTATE, ECUDA, ENOMEM = 0, -1, -2, -3, -4, -5, -6, -7
PARALLEL_ASYNC, SERIAL_SYNC, PARALLEL_SINGLE_STREAM = 0, 1, 2
POLICIES = {"parallel": PARALLEL_ASYNC, "serial": SERIAL_SYNC, "single_stream": PARALLEL_SINGLE_STREAM}
BACKEND_CUDA, BACKEND_RECORD = 0, 1
R, W, RW = 1, 2, 3
K_I32, K_I64, K_CONST, K_INOUT, K_OUT, K_F32, K_F64 = 0, 1, 2, 3, 4, 5, 6
OPS = {1: "launch", 2: "record", 3: "wait", 4: "h2d", 5: "d2h", 6: "event_sync",
       7: "stream_sync", 8: "wait_copy"}


class DagrtError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"dagrt error {status}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("policy", C.c_int32), ("prefetch", C.c_int32), ("max_streams", C.c_int32),
                ("record_dag", C.c_int32), ("backend", C.c_int32), ("graph_cache", C.c_int32)]


class Dim3(C.Structure):
    _fields_ = [("x", C.c_uint32), ("y", C.c_uint32), ("z", C.c_uint32)]


class LaunchConfig(C.Structure):
    _fields_ = [("grid", Dim3), ("block", Dim3), ("smem", C.c_uint32)]


class Arg(C.Union):
    _fields_ = [("array", C.c_uint64), ("i32", C.c_int32), ("i64", C.c_int64),
                ("f32", C.c_float), ("f64", C.c_double)]


class LaunchDesc(C.Structure):
    """dagrt_launch_desc (include/dagrt.h)."""
    _fields_ = [("kernel", C.c_uint32), ("grid", Dim3), ("block", Dim3), ("smem", C.c_uint32),
                ("nargs", C.c_int32), ("args", C.POINTER(Arg))]


class VertexInfo(C.Structure):
    _fields_ = [("id", C.c_uint32), ("kind", C.c_uint32), ("kernel", C.c_uint32),
                ("stream", C.c_int32), ("array", C.c_uint64)]


class EdgeInfo(C.Structure):
    _fields_ = [("parent", C.c_uint32), ("child", C.c_uint32), ("array", C.c_uint64)]


class TraceOp(C.Structure):
    _fields_ = [("op", C.c_int32), ("stream", C.c_int32), ("a", C.c_int64), ("b", C.c_int64),
                ("bytes", C.c_uint64)]


STAT_FIELDS = ["launches", "vertices", "host_vertices", "edges", "cross_stream_waits",
               "copy_waits", "streams", "events_created", "h2d_bytes", "d2h_bytes",
               "h2d_copies", "d2h_copies", "host_syncs", "sched_ns", "graph_replays",
               "graph_captures", "eager_batches", "launch_ns", "record_ns", "wait_ns",
               "table_vertices", "epoch_base", "max_readers", "um_prefetch_bytes", "um_fault_bytes"]


class Stats(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in STAT_FIELDS]


_lib = None
_fast = False


def fast():
    """The CPython fastcall module over libdagrt.so (pyext/dagrt_fastcall.c),
    or None if it was not built: the same C calls, without ctypes' ~1-2 us of
    argument marshalling per call."""
    global _fast
    if _fast is False:
        lib()
        try:
            from . import _dagrt_fastcall as m
        except ImportError:
            m = None
        _fast = m
    return _fast


def lib():
    """Load libdagrt.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIBPATH):
        raise ImportError(f"{LIBPATH} not built: run `python -m paper_2012_09646_b200.build`")
    L = C.CDLL(LIBPATH)
    st = C.c_int32
    ctx = C.c_void_p
    L.dagrt_create.argtypes = [C.c_int, C.POINTER(Config), C.POINTER(C.c_void_p)]
    L.dagrt_destroy.argtypes = [ctx]
    L.dagrt_last_error.argtypes = [ctx]
    L.dagrt_last_error.restype = C.c_char_p
    L.dagrt_array_register.argtypes = [ctx, C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_uint64)]
    L.dagrt_array_unregister.argtypes = [ctx, C.c_uint64]
    L.dagrt_array_device_ptr.argtypes = [ctx, C.c_uint64, C.POINTER(C.c_void_p)]
    L.dagrt_kernel_register.argtypes = [ctx, C.c_void_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_uint32)]
    L.dagrt_kernel_lookup.argtypes = [ctx, C.c_char_p, C.POINTER(C.c_uint32)]
    L.dagrt_kernel_signature.argtypes = [ctx, C.c_uint32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.dagrt_builtin_count.restype = C.c_int32
    L.dagrt_builtin_name.argtypes = [C.c_int32]
    L.dagrt_builtin_name.restype = C.c_char_p
    L.dagrt_builtin_signature.argtypes = [C.c_int32]
    L.dagrt_builtin_signature.restype = C.c_char_p
    L.dagrt_launch.argtypes = [ctx, C.c_uint32, Dim3, Dim3, C.c_uint32, C.POINTER(Arg), C.c_int32]
    L.dagrt_launch_raw.argtypes = [ctx, C.c_uint32, Dim3, Dim3, C.c_uint32, C.POINTER(Arg), C.c_int32,
                                   C.c_void_p]
    L.dagrt_launch_prepared.argtypes = [ctx, C.c_void_p]
    L.dagrt_launch_batch.argtypes = [ctx, C.c_void_p, C.c_int32]
    L.dagrt_host_read.argtypes = [ctx, C.c_uint64, C.c_size_t, C.c_size_t, C.c_void_p]
    L.dagrt_host_write.argtypes = [ctx, C.c_uint64, C.c_size_t, C.c_size_t, C.c_void_p]
    L.dagrt_host_map.argtypes = [ctx, C.c_uint64, C.c_int32, C.POINTER(C.c_void_p)]
    L.dagrt_host_unmap.argtypes = [ctx, C.c_uint64]
    L.dagrt_sync.argtypes = [ctx]
    L.dagrt_dag_export.argtypes = [ctx, C.POINTER(VertexInfo), C.POINTER(C.c_uint32),
                                   C.POINTER(EdgeInfo), C.POINTER(C.c_uint32)]
    L.dagrt_dag_clear.argtypes = [ctx]
    L.dagrt_trace_export.argtypes = [ctx, C.POINTER(TraceOp), C.POINTER(C.c_uint32)]
    L.dagrt_stats.argtypes = [ctx, C.c_void_p, C.c_size_t]
    L.dagrt_stats_reset.argtypes = [ctx]
    L.dagrt_stream_count.argtypes = [ctx, C.POINTER(C.c_int32)]
    L.dagrt_stream_handle.argtypes = [ctx, C.c_int32, C.POINTER(C.c_void_p)]
    L.dagrt_profile_enable.argtypes = [ctx, C.c_uint32, C.c_int32]
    L.dagrt_profile_collect.argtypes = [ctx, C.c_uint32, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.dagrt_graph_create.argtypes = [ctx, C.POINTER(C.c_void_p)]
    L.dagrt_graph_add_kernel.argtypes = [ctx, C.c_void_p, C.c_uint32, Dim3, Dim3, C.c_uint32,
                                         C.POINTER(Arg), C.c_int32, C.POINTER(C.c_uint32), C.c_int32,
                                         C.POINTER(C.c_uint32)]
    L.dagrt_graph_add_copy.argtypes = [ctx, C.c_void_p, C.c_uint64, C.c_int32, C.c_size_t, C.c_size_t,
                                       C.POINTER(C.c_uint32), C.c_int32, C.POINTER(C.c_uint32)]
    L.dagrt_graph_add_read.argtypes = [ctx, C.c_void_p, C.c_uint64, C.c_size_t, C.c_size_t, C.c_void_p,
                                       C.POINTER(C.c_uint32), C.c_int32, C.POINTER(C.c_uint32)]
    L.dagrt_graph_instantiate.argtypes = [ctx, C.c_void_p]
    L.dagrt_graph_run.argtypes = [ctx, C.c_void_p, C.c_int32]
    L.dagrt_graph_destroy.argtypes = [ctx, C.c_void_p]
    for name in dir(L):
        pass
    for fn in ("dagrt_create", "dagrt_destroy", "dagrt_array_register", "dagrt_array_unregister",
               "dagrt_array_device_ptr", "dagrt_kernel_register", "dagrt_kernel_lookup",
               "dagrt_kernel_signature", "dagrt_launch", "dagrt_launch_prepared", "dagrt_launch_batch",
               "dagrt_launch_raw",
               "dagrt_host_read",
               "dagrt_host_write", "dagrt_host_map", "dagrt_host_unmap", "dagrt_sync",
               "dagrt_dag_export", "dagrt_dag_clear", "dagrt_trace_export", "dagrt_stats",
               "dagrt_stats_reset", "dagrt_stream_count", "dagrt_stream_handle",
               "dagrt_profile_enable", "dagrt_profile_collect",
               "dagrt_graph_create", "dagrt_graph_add_kernel", "dagrt_graph_add_copy",
               "dagrt_graph_add_read", "dagrt_graph_instantiate", "dagrt_graph_run", "dagrt_graph_destroy"):
        getattr(L, fn).restype = st
    _lib = L
    return L


EXP_LIBPATH = os.path.join(HERE, "libdagrt_exp.so")
_exp = None


def load_experimental():
    """Load libdagrt_exp.so (csrc/exp/): the measured-but-not-shipped kernel
    variants (round-1 kernels, tuning shapes) register into the built-in
    registry; contexts find them by name (dagrt_kernel_lookup).  Tests and
    tools only -- the product path never loads it."""
    global _exp
    if _exp is None:
        lib()  # the registry lives in libdagrt.so, the exp library's dependency
        if not os.path.exists(EXP_LIBPATH):
            raise ImportError(f"{EXP_LIBPATH} not built: run `python -m paper_2012_09646_b200.build`")
        _exp = C.CDLL(EXP_LIBPATH)
    return _exp


def managed_alloc(nbytes):
    """cudaMallocManaged through the library (dagrt_managed_alloc)."""
    L = lib()
    L.dagrt_managed_alloc.argtypes = [C.c_size_t, C.POINTER(C.c_void_p)]
    L.dagrt_managed_alloc.restype = C.c_int32
    p = C.c_void_p()
    s = L.dagrt_managed_alloc(nbytes, C.byref(p))
    if s:
        raise DagrtError(s, f"cudaMallocManaged({nbytes}) failed")
    return p.value


def managed_free(ptr):
    L = lib()
    L.dagrt_managed_free.argtypes = [C.c_void_p]
    L.dagrt_managed_free(C.c_void_p(ptr))


def managed_to_host(ptr, nbytes):
    """Move the pages of a managed range to the host (dagrt_managed_to_host)."""
    L = lib()
    L.dagrt_managed_to_host.argtypes = [C.c_void_p, C.c_size_t]
    L.dagrt_managed_to_host.restype = C.c_int32
    s = L.dagrt_managed_to_host(C.c_void_p(ptr), nbytes)
    if s:
        raise DagrtError(s, "managed prefetch to host failed")


def builtins():
    L = lib()
    return [(L.dagrt_builtin_name(i).decode(), L.dagrt_builtin_signature(i).decode())
            for i in range(L.dagrt_builtin_count())]


def dim3(v):
    if isinstance(v, str) and v == "auto":  # history-driven launch configuration (dagrt_kernel_autotune)
        return Dim3(0, 0, 0)
    if isinstance(v, int):
        return Dim3(v, 1, 1)
    v = tuple(v) + (1, 1)
    return Dim3(v[0], v[1], v[2])


class Array:
    """A registered array.  Keeps the caller's tensors alive until unregister."""
    __slots__ = ("ctx", "handle", "name", "nbytes", "dev_ptr", "host_ptr", "_keep")

    def __init__(self, ctx, handle, name, nbytes, dev_ptr, host_ptr, keep):
        self.ctx, self.handle, self.name, self.nbytes = ctx, handle, name, nbytes
        self.dev_ptr, self.host_ptr, self._keep = dev_ptr, host_ptr, keep

    def __repr__(self):
        return f"Array({self.name}, {self.nbytes} B)"


class Kernel:
    __slots__ = ("handle", "name", "kinds")

    def __init__(self, handle, name, kinds):
        self.handle, self.name, self.kinds = handle, name, kinds


def _set_arg(slot, kind, v):
    if K_CONST <= kind <= K_OUT:
        if not isinstance(v, Array):
            raise TypeError(f"pointer parameter needs an Array, got {type(v)}")
        slot.array = v.handle
    elif kind == K_I32:
        slot.i64 = 0
        slot.i32 = int(v)
    elif kind == K_I64:
        slot.i64 = int(v)
    elif kind == K_F32:
        slot.i64 = 0
        slot.f32 = float(v)
    elif kind == K_F64:
        slot.f64 = float(v)
    else:
        raise ValueError(kind)


class Launch:
    """A prepared launch (args marshalled once; calling it enqueues it)."""
    __slots__ = ("ctx", "kernel", "grid", "block", "smem", "args", "n", "_fn", "_c", "_desc", "_dp")

    def __init__(self, ctx, kernel, grid, block, args, smem=0):
        if len(args) != len(kernel.kinds):
            raise DagrtError(ESIG, f"{kernel.name}: {len(args)} args, signature has {len(kernel.kinds)}")
        self.ctx, self.kernel, self.smem = ctx, kernel, smem
        self.grid, self.block = dim3(grid), dim3(block)
        self.n = len(args)
        self.args = (Arg * max(1, self.n))()
        for i, (k, v) in enumerate(zip(kernel.kinds, args)):
            _set_arg(self.args[i], k, v)
        # one descriptor per prepared launch: each call passes two pointers
        # (dagrt_launch_prepared) instead of marshalling seven arguments
        self._desc = LaunchDesc(kernel.handle, self.grid, self.block, smem, self.n, self.args)
        self._dp = C.addressof(self._desc)
        self._fn = lib().dagrt_launch_prepared
        self._c = ctx._c

    def __call__(self):
        s = self._fn(self._c, self._dp)
        if s:
            self.ctx._raise(s)

    def raw(self, stream_ptr):
        s = lib().dagrt_launch_raw(self._c, self.kernel.handle, self.grid, self.block, self.smem,
                                   self.args, self.n, C.c_void_p(stream_ptr))
        if s:
            self.ctx._raise(s)


class Batch:
    """Prepared launches issued in program order by ONE call
    (dagrt_launch_batch): the same DAG, streams and events as calling each
    Launch in turn, one Python->C transition instead of len(launches)."""
    __slots__ = ("ctx", "launches", "_arr", "_n", "_fn", "_c", "_p")

    def __init__(self, ctx, launches):
        self.ctx, self.launches = ctx, list(launches)
        self._n = len(self.launches)
        self._arr = (LaunchDesc * max(1, self._n))()
        for i, L in enumerate(self.launches):
            C.memmove(C.byref(self._arr, i * C.sizeof(LaunchDesc)), L._dp, C.sizeof(LaunchDesc))
        self._p = C.addressof(self._arr)
        self._c = ctx._c
        f = fast()
        if f is not None:  # functools.partial: no Python frame per call
            self._fn = functools.partial(f.launch_batch, ctx._c.value, self._p, self._n)
        else:
            self._fn = functools.partial(lib().dagrt_launch_batch, ctx._c, self._p, self._n)

    def __call__(self):
        s = self._fn()
        if s:
            self.ctx._raise(s)


class Graph:
    """Hand-built CUDA graph with manual dependencies (baseline, L1062-1067)."""

    def __init__(self, ctx):
        self.ctx = ctx
        h = C.c_void_p()
        ctx._check(lib().dagrt_graph_create(ctx._c, C.byref(h)))
        self._h = h

    def _deps(self, deps):
        deps = list(deps or [])
        return (C.c_uint32 * max(1, len(deps)))(*deps), len(deps)

    def kernel(self, launch: Launch, deps=()):
        d, nd = self._deps(deps)
        node = C.c_uint32()
        self.ctx._check(lib().dagrt_graph_add_kernel(
            self.ctx._c, self._h, launch.kernel.handle, launch.grid, launch.block, launch.smem,
            launch.args, launch.n, d, nd, C.byref(node)))
        return node.value

    def copy(self, arr: Array, direction, off=0, nbytes=None, deps=()):
        d, nd = self._deps(deps)
        node = C.c_uint32()
        nb = arr.nbytes - off if nbytes is None else nbytes
        self.ctx._check(lib().dagrt_graph_add_copy(self.ctx._c, self._h, arr.handle,
                                                   0 if direction == "h2d" else 1, off, nb, d, nd,
                                                   C.byref(node)))
        return node.value

    def read(self, arr: Array, dst_ptr, off=0, nbytes=4, deps=()):
        """D2H node into caller-owned pinned host memory at address dst_ptr."""
        d, nd = self._deps(deps)
        node = C.c_uint32()
        self.ctx._check(lib().dagrt_graph_add_read(self.ctx._c, self._h, arr.handle, off, nbytes,
                                                   C.c_void_p(dst_ptr), d, nd, C.byref(node)))
        return node.value

    def instantiate(self):
        self.ctx._check(lib().dagrt_graph_instantiate(self.ctx._c, self._h))

    def run(self, wait=True):
        f = fast()
        if f is not None:  # same binding speed as the scheduler's batch/read calls
            s = f.graph_run(self.ctx._c.value, self._h.value, 1 if wait else 0)
        else:
            s = lib().dagrt_graph_run(self.ctx._c, self._h, 1 if wait else 0)
        if s:
            self.ctx._raise(s)


class Context:
    def __init__(self, device=0, policy="parallel", prefetch=True, max_streams=0,
                 record_dag=False, backend="cuda", graph_cache=False):
        L = lib()
        cfg = Config(POLICIES[policy], 1 if prefetch else 0,
                     max_streams, 1 if record_dag else 0,
                     BACKEND_CUDA if backend == "cuda" else BACKEND_RECORD, 1 if graph_cache else 0)
        h = C.c_void_p()
        s = L.dagrt_create(device, C.byref(cfg), C.byref(h))
        if s:
            raise DagrtError(s, "dagrt_create failed (CUDA device unavailable?)")
        self._c = h
        self.policy, self.backend = policy, backend
        self.arrays = {}      # handle -> Array
        self._kernels = {}
        self._kname = {}      # kernel handle -> name

    # -- errors
    def _raise(self, s):
        raise DagrtError(s, lib().dagrt_last_error(self._c).decode())

    def _check(self, s):
        if s:
            self._raise(s)

    @classmethod
    def _borrow(cls, handle, policy="parallel", backend="cuda"):
        """A view of a context owned elsewhere (a multi-context's slot)."""
        self = cls.__new__(cls)
        self._c = C.c_void_p(handle)
        self.policy, self.backend = policy, backend
        self.arrays, self._kernels, self._kname = {}, {}, {}
        self._borrowed = True
        return self

    def close(self):
        if self._c and not getattr(self, "_borrowed", False):
            lib().dagrt_destroy(self._c)
        self._c = None
        self.arrays.clear()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- arrays
    def register(self, name, dev_ptr, nbytes, host_ptr=None, keep=()):
        h = C.c_uint64()
        self._check(lib().dagrt_array_register(self._c, C.c_void_p(dev_ptr),
                                               C.c_void_p(host_ptr) if host_ptr else None,
                                               nbytes, C.byref(h)))
        a = Array(self, h.value, name, nbytes, dev_ptr, host_ptr, keep)
        self.arrays[a.handle] = a
        return a

    def register_managed(self, name, ptr, nbytes, keep=()):
        """Unified-memory array (dagrt_array_register_managed: the UM mode)."""
        L = lib()
        L.dagrt_array_register_managed.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_uint64)]
        L.dagrt_array_register_managed.restype = C.c_int32
        h = C.c_uint64()
        self._check(L.dagrt_array_register_managed(self._c, C.c_void_p(ptr), nbytes, C.byref(h)))
        a = Array(self, h.value, name, nbytes, ptr, ptr, keep)
        self.arrays[a.handle] = a
        return a

    def register_tensor(self, name, t, mirror=None):
        """Register a device tensor (and optional pinned host mirror tensor)."""
        nbytes = t.numel() * t.element_size()
        if mirror is not None:
            assert mirror.numel() * mirror.element_size() == nbytes
        return self.register(name, t.data_ptr(), nbytes,
                             mirror.data_ptr() if mirror is not None else None, keep=(t, mirror))

    def unregister(self, a: Array):
        self._check(lib().dagrt_array_unregister(self._c, a.handle))
        self.arrays.pop(a.handle, None)

    # -- kernels
    def kernel(self, name):
        k = self._kernels.get(name)
        if k is not None:
            return k
        L = lib()
        h = C.c_uint32()
        self._check(L.dagrt_kernel_lookup(self._c, name.encode(), C.byref(h)))
        n = C.c_int32(16)
        kinds = (C.c_int32 * 16)()
        self._check(L.dagrt_kernel_signature(self._c, h.value, kinds, C.byref(n)))
        k = Kernel(h.value, name, list(kinds[:n.value]))
        self._kernels[name] = k
        self._kname[h.value] = name
        return k

    def register_kernel(self, fn_ptr, name, signature):
        h = C.c_uint32()
        self._check(lib().dagrt_kernel_register(self._c, C.c_void_p(fn_ptr), name.encode(),
                                                signature.encode(), C.byref(h)))
        self._kernels.pop(name, None)
        return self.kernel(name)

    def prepare(self, kernel, grid, block, args, smem=0):
        if isinstance(kernel, str):
            kernel = self.kernel(kernel)
        return Launch(self, kernel, grid, block, args, smem)

    def launch(self, kernel, grid, block, *args, smem=0):
        self.prepare(kernel, grid, block, args, smem)()

    def autotune(self, kernel, candidates, trials=3):
        """Candidate (grid, block, smem) configurations for launches of
        `kernel` with grid "auto" (dagrt_kernel_autotune)."""
        k = self.kernel(kernel) if isinstance(kernel, str) else kernel
        arr = (LaunchConfig * len(candidates))()
        for i, cand in enumerate(candidates):
            g, b = cand[0], cand[1]
            sm = cand[2] if len(cand) > 2 else 0
            arr[i] = LaunchConfig(dim3(g), dim3(b), sm)
        L = lib()
        L.dagrt_kernel_autotune.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_int32, C.c_int32]
        L.dagrt_kernel_autotune.restype = C.c_int32
        self._check(L.dagrt_kernel_autotune(self._c, k.handle, C.addressof(arr), len(candidates), trials))

    def autotune_state(self, kernel):
        """(chosen candidate or -1, [median ms per candidate or -1])."""
        k = self.kernel(kernel) if isinstance(kernel, str) else kernel
        L = lib()
        L.dagrt_autotune_state.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.dagrt_autotune_state.restype = C.c_int32
        ch, n = C.c_int32(), C.c_int32(16)
        ms = (C.c_double * 16)()
        self._check(L.dagrt_autotune_state(self._c, k.handle, C.byref(ch), ms, C.byref(n)))
        return ch.value, list(ms[:n.value])

    LIBFN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p)

    def launch_library(self, fn, name, arrays, modes):
        """A library call as a DAG vertex (dagrt_launch_library): fn(stream)
        is called with the CUDA stream (an int handle) the scheduler picked
        and must enqueue its GPU work there; arrays/modes declare its accesses
        (R, W, RW)."""
        def tramp(stream, _user):
            try:
                fn(stream or 0)
                return 0
            except Exception:  # surfaced as DAGRT_EINVAL
                import traceback
                traceback.print_exc()
                return 1
        cb = self.LIBFN(tramp)
        self._keep = getattr(self, "_keep", [])
        self._keep.append(cb)
        n = len(arrays)
        A = (C.c_uint64 * max(1, n))(*[a.handle for a in arrays])
        M = (C.c_int32 * max(1, n))(*modes)
        L = lib()
        L.dagrt_launch_library.argtypes = [C.c_void_p, self.LIBFN, C.c_void_p, C.c_char_p, C.c_void_p, C.c_void_p,
                                           C.c_int32]
        L.dagrt_launch_library.restype = C.c_int32
        self._check(L.dagrt_launch_library(self._c, cb, None, name.encode(), C.addressof(A), C.addressof(M), n))
        self._kname.setdefault(self._lib_handle(name), name)

    def _lib_handle(self, name):
        k = C.c_uint32()
        if lib().dagrt_kernel_lookup(self._c, name.encode(), C.byref(k)) == 0:
            return k.value
        return -1

    def batch(self, launches):
        """Prepared launches -> one callable that issues them in order (Batch)."""
        return Batch(self, launches)

    # -- host access
    def host_read(self, a: Array, dst_ptr, off=0, nbytes=None):
        nb = a.nbytes - off if nbytes is None else nbytes
        self._check(lib().dagrt_host_read(self._c, a.handle, off, nb, C.c_void_p(dst_ptr)))

    def prepare_read(self, a: Array, dst_ptr, off=0, nbytes=None):
        """A host read with its arguments converted once: calling the result
        is dagrt_host_read(a, off, nbytes, dst) (same semantics as host_read)."""
        nb = a.nbytes - off if nbytes is None else nbytes
        f = fast()
        if f is not None:
            call = functools.partial(f.host_read, self._c.value, a.handle, off, nb, dst_ptr)
        else:
            call = functools.partial(lib().dagrt_host_read, self._c, C.c_uint64(a.handle),
                                     C.c_size_t(off), C.c_size_t(nb), C.c_void_p(dst_ptr))
        raise_ = self._raise

        def read():
            s = call()
            if s:
                raise_(s)
        read.call = call  # the bare call (returns the status)
        return read

    def host_write(self, a: Array, src_ptr, off=0, nbytes=None):
        nb = a.nbytes - off if nbytes is None else nbytes
        self._check(lib().dagrt_host_write(self._c, a.handle, off, nb, C.c_void_p(src_ptr)))

    def read_scalar(self, a: Array, ctype=C.c_float, index=0):
        v = ctype()
        self.host_read(a, C.addressof(v), off=index * C.sizeof(ctype), nbytes=C.sizeof(ctype))
        return v.value

    def host_map(self, a: Array, access=R):
        p = C.c_void_p()
        self._check(lib().dagrt_host_map(self._c, a.handle, access, C.byref(p)))
        return p.value

    def host_unmap(self, a: Array):
        self._check(lib().dagrt_host_unmap(self._c, a.handle))

    def sync(self):
        self._check(lib().dagrt_sync(self._c))

    # -- introspection
    def dag(self):
        """(vertices, edges): vertices = [(id, kind, name, stream)], edges = {(p, c, array_name)}."""
        L = lib()
        nv, ne = C.c_uint32(0), C.c_uint32(0)
        self._check(L.dagrt_dag_export(self._c, None, C.byref(nv), None, C.byref(ne)))
        V = (VertexInfo * max(1, nv.value))()
        E = (EdgeInfo * max(1, ne.value))()
        self._check(L.dagrt_dag_export(self._c, V, C.byref(nv), E, C.byref(ne)))
        names = dict(self._kname)
        L.dagrt_kernel_name.argtypes = [C.c_void_p, C.c_uint32]
        L.dagrt_kernel_name.restype = C.c_char_p
        for v in V[:nv.value]:
            if v.kind == 0 and v.kernel not in names:
                nm = L.dagrt_kernel_name(self._c, v.kernel)
                if nm:
                    names[v.kernel] = nm.decode()
        arr = {h: a.name for h, a in self.arrays.items()}
        verts = []
        for v in V[:nv.value]:
            if v.kind == 0:
                verts.append((v.id, "kernel", names.get(v.kernel, f"k{v.kernel}"), v.stream))
            else:
                verts.append((v.id, "host", arr.get(v.array, hex(v.array)), -1))
        edges = {(e.parent, e.child, arr.get(e.array, hex(e.array))) for e in E[:ne.value]}
        return verts, edges

    def dag_clear(self):
        self._check(lib().dagrt_dag_clear(self._c))

    def trace(self):
        L = lib()
        n = C.c_uint32(0)
        self._check(L.dagrt_trace_export(self._c, None, C.byref(n)))
        T = (TraceOp * max(1, n.value))()
        self._check(L.dagrt_trace_export(self._c, T, C.byref(n)))
        return [(OPS[t.op], t.stream, t.a, t.b, t.bytes) for t in T[:n.value]]

    def stats(self):
        s = Stats()
        self._check(lib().dagrt_stats(self._c, C.byref(s), C.sizeof(s)))
        return {f: getattr(s, f) for f in STAT_FIELDS}

    def stats_reset(self):
        self._check(lib().dagrt_stats_reset(self._c))

    def stream_count(self):
        n = C.c_int32()
        self._check(lib().dagrt_stream_count(self._c, C.byref(n)))
        return n.value

    def stream_handle(self, i):
        p = C.c_void_p()
        self._check(lib().dagrt_stream_handle(self._c, i, C.byref(p)))
        return p.value

    def graph(self):
        return Graph(self)

    def profile(self, kernel, on=True):
        k = self.kernel(kernel) if isinstance(kernel, str) else kernel
        self._check(lib().dagrt_profile_enable(self._c, k.handle, 1 if on else 0))

    def profile_collect(self, kernel):
        """(launches, sum of launch ms, busy ms = union of launch intervals)."""
        k = self.kernel(kernel) if isinstance(kernel, str) else kernel
        n, s, b = C.c_int32(), C.c_double(), C.c_double()
        self._check(lib().dagrt_profile_collect(self._c, k.handle, C.byref(n), C.byref(s), C.byref(b)))
        return n.value, s.value, b.value


class TimelineRec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("stream", C.c_int32), ("vertex", C.c_int64), ("id", C.c_int64),
                ("bytes", C.c_uint64), ("start_ms", C.c_double), ("end_ms", C.c_double)]


def _timeline_enable(self, on=True):
    L = lib()
    L.dagrt_timeline_enable.argtypes = [C.c_void_p, C.c_int32]
    L.dagrt_timeline_enable.restype = C.c_int32
    self._check(L.dagrt_timeline_enable(self._c, 1 if on else 0))


def _timeline_export(self):
    """[(kind, stream, vertex, id, bytes, start_ms, end_ms)]; kind 'kernel'|'h2d'|'d2h'."""
    L = lib()
    L.dagrt_timeline_export.argtypes = [C.c_void_p, C.POINTER(TimelineRec), C.POINTER(C.c_uint32)]
    L.dagrt_timeline_export.restype = C.c_int32
    n = C.c_uint32(0)
    self._check(L.dagrt_timeline_export(self._c, None, C.byref(n)))
    R = (TimelineRec * max(1, n.value))()
    self._check(L.dagrt_timeline_export(self._c, R, C.byref(n)))
    kinds = {0: "kernel", 1: "h2d", 2: "d2h"}
    return [(kinds[r.kind], r.stream, r.vertex, r.id, r.bytes, r.start_ms, r.end_ms) for r in R[:n.value]]


Context.timeline = _timeline_enable
Context.timeline_export = _timeline_export


# ---------------------------------------------------------------- multi-GPU placement (f2)

class MultiStats(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("migrations_peer", C.c_uint64), ("bytes_peer", C.c_uint64),
                ("migrations_host", C.c_uint64), ("bytes_host", C.c_uint64), ("replicas", C.c_uint64),
                ("bytes_replicas", C.c_uint64), ("per_slot", C.c_uint64 * 16)]


class MultiArray:
    """A multi-array (dagrt_marray): home copy, library-owned replicas, optional mirror."""
    __slots__ = ("multi", "handle", "name", "nbytes", "host_ptr", "_keep")

    def __init__(self, multi, handle, name, nbytes, host_ptr, keep):
        self.multi, self.handle, self.name, self.nbytes = multi, handle, name, nbytes
        self.host_ptr, self._keep = host_ptr, keep

    def __repr__(self):
        return f"MultiArray({self.name}, {self.nbytes} B)"


PLACEMENTS = {"data": 0, "round_robin": 1}


def _multi_lib():
    L = lib()
    if getattr(L, "_multi_ready", False):
        return L
    vp, st = C.c_void_p, C.c_int32
    L.dagrt_multi_create.argtypes = [C.POINTER(C.c_int32), C.c_int32, C.POINTER(Config), C.c_int32, C.POINTER(vp)]
    L.dagrt_multi_destroy.argtypes = [vp]
    L.dagrt_multi_last_error.argtypes = [vp]
    L.dagrt_multi_last_error.restype = C.c_char_p
    L.dagrt_multi_slot_ctx.argtypes = [vp, C.c_int32, C.POINTER(vp)]
    L.dagrt_multi_array_register.argtypes = [vp, C.c_int32, vp, vp, C.c_size_t, C.POINTER(C.c_uint64)]
    L.dagrt_multi_array_ptr.argtypes = [vp, C.c_uint64, C.c_int32, C.POINTER(vp)]
    L.dagrt_multi_launch.argtypes = [vp, C.c_char_p, Dim3, Dim3, C.c_uint32, C.POINTER(Arg), C.c_int32, C.c_int32,
                                     C.POINTER(C.c_int32)]
    L.dagrt_multi_host_read.argtypes = [vp, C.c_uint64, C.c_size_t, C.c_size_t, vp]
    L.dagrt_multi_host_write.argtypes = [vp, C.c_uint64, C.c_size_t, C.c_size_t, vp]
    L.dagrt_multi_sync.argtypes = [vp]
    L.dagrt_multi_stats.argtypes = [vp, C.POINTER(MultiStats)]
    for fn in ("dagrt_multi_create", "dagrt_multi_destroy", "dagrt_multi_slot_ctx", "dagrt_multi_array_register",
               "dagrt_multi_array_ptr", "dagrt_multi_launch", "dagrt_multi_host_read", "dagrt_multi_host_write",
               "dagrt_multi_sync", "dagrt_multi_stats"):
        getattr(L, fn).restype = st
    L._multi_ready = True
    return L


class Multi:
    """Multi-GPU DAG placement (include/dagrt.h "multi-GPU placement", SURVEY
    f2): one scheduler context per slot, launches placed
    by data location and estimated migration cost, cross-slot edges as peer
    copies plus cross-device events.  `devices` lists each slot's CUDA device
    (repeat a device to exercise the cross-slot path on one GPU)."""

    def __init__(self, devices=(0,), placement="data", policy="parallel", prefetch=True, max_streams=0,
                 record_dag=False, backend="cuda", graph_cache=False):
        L = _multi_lib()
        n = len(devices)
        devs = (C.c_int32 * n)(*devices)
        cfg = Config(POLICIES[policy], 1 if prefetch else 0, max_streams, 1 if record_dag else 0,
                     BACKEND_CUDA if backend == "cuda" else BACKEND_RECORD, 1 if graph_cache else 0)
        h = C.c_void_p()
        s = L.dagrt_multi_create(devs, n, C.byref(cfg), PLACEMENTS[placement], C.byref(h))
        if s:
            raise DagrtError(s, "dagrt_multi_create failed")
        self._m, self.devices, self.backend, self.policy = h, list(devices), backend, policy
        self.arrays = {}
        self._kinds = {}

    def _check(self, s):
        if s:
            raise DagrtError(s, _multi_lib().dagrt_multi_last_error(self._m).decode())

    def close(self):
        if self._m:
            _multi_lib().dagrt_multi_destroy(self._m)
            self._m = None
            self.arrays.clear()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def register(self, name, nbytes, home=0, dev_ptr=None, host_ptr=None, keep=()):
        h = C.c_uint64()
        self._check(_multi_lib().dagrt_multi_array_register(self._m, home, C.c_void_p(dev_ptr) if dev_ptr else None,
                                                             C.c_void_p(host_ptr) if host_ptr else None, nbytes,
                                                             C.byref(h)))
        a = MultiArray(self, h.value, name, nbytes, host_ptr, keep)
        self.arrays[a.handle] = a
        return a

    def register_tensor(self, name, t=None, home=0, mirror=None):
        """Device tensor t on slot `home` (None: the library allocates the home
        copy) and/or a pinned host mirror tensor."""
        ref = t if t is not None else mirror
        nbytes = ref.numel() * ref.element_size()
        return self.register(name, nbytes, home, t.data_ptr() if t is not None else None,
                             mirror.data_ptr() if mirror is not None else None, keep=(t, mirror))

    def ptr(self, a, slot):
        p = C.c_void_p()
        self._check(_multi_lib().dagrt_multi_array_ptr(self._m, a.handle, slot, C.byref(p)))
        return p.value

    def slot_context(self, slot):
        """The slot's own scheduler context (borrowed: DAG export, stats)."""
        p = C.c_void_p()
        self._check(_multi_lib().dagrt_multi_slot_ctx(self._m, slot, C.byref(p)))
        return Context._borrow(p.value, self.policy, self.backend)

    def _signature(self, name):
        k = self._kinds.get(name)
        if k is None:
            ctx = self.slot_context(0)
            k = ctx.kernel(name).kinds
            self._kinds[name] = k
        return k

    def launch(self, name, grid, block, *args, smem=0, slot=-1):
        """Launch `name`; returns the slot it was placed on."""
        kinds = self._signature(name)
        if len(args) != len(kinds):
            raise DagrtError(ESIG, f"{name}: {len(args)} args, signature has {len(kinds)}")
        A = (Arg * max(1, len(args)))()
        for i, (k, v) in enumerate(zip(kinds, args)):
            if K_CONST <= k <= K_OUT:
                if not isinstance(v, MultiArray):
                    raise TypeError(f"pointer parameter needs a MultiArray, got {type(v)}")
                A[i].array = v.handle
            else:
                _set_arg(A[i], k, v)
        placed = C.c_int32(-1)
        self._check(_multi_lib().dagrt_multi_launch(self._m, name.encode(), dim3(grid), dim3(block), smem, A,
                                                     len(args), slot, C.byref(placed)))
        return placed.value

    def read(self, a, dst_ptr, off=0, nbytes=None):
        n = a.nbytes - off if nbytes is None else nbytes
        self._check(_multi_lib().dagrt_multi_host_read(self._m, a.handle, off, n, C.c_void_p(dst_ptr)))

    def write(self, a, src_ptr, off=0, nbytes=None):
        n = a.nbytes - off if nbytes is None else nbytes
        self._check(_multi_lib().dagrt_multi_host_write(self._m, a.handle, off, n, C.c_void_p(src_ptr)))

    def sync(self):
        self._check(_multi_lib().dagrt_multi_sync(self._m))

    def stats(self):
        s = MultiStats()
        self._check(_multi_lib().dagrt_multi_stats(self._m, C.byref(s)))
        d = {f: getattr(s, f) for f, _ in MultiStats._fields_ if f != "per_slot"}
        d["per_slot"] = list(s.per_slot[:len(self.devices)])
        return d
