"""Common scaffolding of the benchmark host programs.

A program owns its device tensors (torch, for memory only), registers them
with a dagrt Context, and exposes ``run()``: the benchmark's host code written
sequentially, as the paper's users write it -- kernel
launches followed by host reads of the sinks, with no streams or events in
sight.  The same ``run()`` executes under the parallel-async scheduler and
under the serial-sync policy (the GrCUDA baseline, L559-569).  ``graph()``
builds the hand-written CUDA Graph baseline (manual dependencies, L1062-1067).

Modes:
* ``resident`` -- inputs are device-valid before the run; the host reads one
  element of each sink (the ``Z[0]`` pattern of Fig. 4);
* ``stream``   -- inputs are rewritten by the host before every run (host
  newer => H2D inside the run, overlapped by the prefetcher, L356-366) and the
  host reads whole sink arrays (D2H inside the run).
* ``um``       -- the stream workload on UNIFIED memory (GrCUDA's managed
  arrays, §V-C): every array is cudaMallocManaged, the
  inputs' pages are moved to the host before each run (restart(), outside
  the timed region: the host rewrote them), the run either prefetches them
  (context prefetch on: cudaMemPrefetchAsync) or leaves them to GPU page
  faults (prefetch off), and the host maps whole sinks in place (with
  prefetch on, the runtime moves them to the host first).
"""
from __future__ import annotations

import ctypes as C
import weakref

import torch

import synth
from .. import dagrt as D

SMS = 148


def grid_1d(n_items, block=256, per_thread=1, waves=8):
    """Grid for a grid-stride kernel: enough CTAs for `n_items`, capped at
    `waves` CTAs per SM (148 SMs)."""
    need = max(1, -(-n_items // (block * per_thread)))
    return int(min(need, SMS * waves))


class Program:
    name = "?"
    red_bytes = 8 + 8 * 1024  # RedOut: float result, counter, 1024 fp64 partials

    def __init__(self, ctx: D.Context, mode="resident", seed=synth.BASE_SEED, device=None,
                 share=None):
        self.ctx = ctx
        self.mode = mode
        self.share = share  # another Program whose tensors this one reuses (baseline runs)
        self.seed = seed
        self.record = ctx.backend == "record"
        self.device = torch.device("cpu") if self.record else (device or torch.device("cuda"))
        self.t = {}        # name -> device tensor
        self.mirror = {}   # name -> pinned host tensor
        self.a = {}        # name -> dagrt.Array
        self.inputs = []   # arrays the host rewrites before every run (stream mode)
        self.sinks = []    # arrays the host reads at the end of every run
        self._scalar = (C.c_char * 8)()
        self.red = set()   # scalar-reduction outputs (the host reads only the result)
        self.um = mode == "um"
        self.streaming = mode in ("stream", "um")  # host-newer inputs, whole-sink reads

    # ---------------------------------------------------------- allocation
    def alloc(self, name, numel, dtype, mirror=False, zero=False, nbytes=None):
        if self.share is not None and name in self.share.t:
            t = self.share.t[name]
            m = self.share.mirror.get(name) if mirror else None
            if mirror and m is None:
                m = torch.empty(t.numel(), dtype=t.dtype, pin_memory=not self.record)
                m.copy_(t.cpu() if self.record else t)
            if m is not None:
                self.mirror[name] = m
            self.t[name] = t
            self.a[name] = self.ctx.register_tensor(name, t, m)
            return t
        if self.um and not self.record:
            return self._alloc_managed(name, numel, dtype, zero, nbytes)
        if nbytes is not None:
            t = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        elif zero:
            t = torch.zeros(numel, dtype=dtype, device=self.device)
        else:
            t = torch.empty(numel, dtype=dtype, device=self.device)
        m = None
        if mirror:
            m = torch.empty(t.numel(), dtype=t.dtype, pin_memory=not self.record)
            self.mirror[name] = m
        self.t[name] = t
        self.a[name] = self.ctx.register_tensor(name, t, m)
        return t

    _TYPESTR = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4", torch.int64: "<i8",
                torch.uint8: "|u1"}

    def _alloc_managed(self, name, numel, dtype, zero, nbytes):
        """UM mode: cudaMallocManaged memory viewed as a CUDA tensor (no copy)."""
        if nbytes is not None:
            numel, dtype, zero = nbytes, torch.uint8, True
        size = max(1, numel) * torch.empty(0, dtype=dtype).element_size()
        ptr = D.managed_alloc(size)
        weakref.finalize(self, D.managed_free, ptr)

        class _View:  # __cuda_array_interface__: torch.as_tensor shares the memory
            __cuda_array_interface__ = {"shape": (numel,), "typestr": self._TYPESTR[dtype],
                                        "data": (ptr, False), "version": 2, "strides": None}
        t = torch.as_tensor(_View(), device="cuda")
        if zero:
            t.zero_()
        self.t[name] = t
        self.a[name] = self.ctx.register_managed(name, ptr, numel * t.element_size(), keep=(t,))
        return t

    def alloc_red(self, name):
        """Scalar-reduction output: RedOut layout (see csrc/kcommon.cuh)."""
        self.red.add(name)
        return self.alloc(name, 0, None, mirror=self.streaming, nbytes=self.red_bytes)

    def fill(self, name, spec, set_index=0):
        """Seeded input (synth) into the device tensor; stream mode: and its mirror."""
        if self.record or (self.share is not None and name in self.share.t
                           and (name not in self.mirror or name in self.share.mirror)):
            return
        import synth.gpu as sg
        sg.fill_tensor(self.t[name].view(-1), self.seed + set_index, name, spec)
        if name in self.mirror:
            self.mirror[name].copy_(self.t[name].view(self.mirror[name].dtype).view(-1))

    def upload(self, name, host_array):
        """Static data written once from the host (weights, graph)."""
        src = torch.from_numpy(host_array).reshape(-1)
        if self.record:
            return
        self.t[name].view(src.dtype).copy_(src)

    def load_inputs(self, set_index=0):
        """Seeded inputs into HBM (and mirrors), then a device-wide sync so
        torch's asynchronous allocations/zero-fills (on torch's stream) are
        complete before any dagrt stream touches the memory."""
        self._inputs(set_index)
        self.settle()

    def _inputs(self, set_index):
        raise NotImplementedError

    def settle(self):
        if not self.record:
            torch.cuda.synchronize()

    # ---------------------------------------------------------- the run
    def restart(self):
        """Host-side preparation of a fresh run, outside the timed region
        (the paper writes the inputs before each run, L862-864): a no-op
        except for programs whose inputs are also their outputs (HITS), and
        in UM mode, where the inputs' pages go back to the host (as if the
        host had rewritten them) so that the run must migrate them again."""
        if self.um and not self.record:
            torch.cuda.synchronize()
            for n in self.inputs:
                D.managed_to_host(self.t[n].data_ptr(), self.t[n].numel() * self.t[n].element_size())

    def begin_run(self):
        """Stream mode: the host writes fresh inputs (host copy becomes newer)."""
        if self.streaming:
            for n in self.inputs:
                self.ctx.host_map(self.a[n], D.W)
                self.ctx.host_unmap(self.a[n])

    def end_run(self):
        """Host reads of the sinks: one element (resident) or whole arrays (stream)."""
        if not self.streaming:
            if getattr(self, "_reads", None) is None:  # arguments converted once
                self._reads = [self.ctx.prepare_read(self.a[n], C.addressof(self._scalar), 0,
                                                     min(4, self.a[n].nbytes)) for n in self.sinks]
            for r in self._reads:
                r()
            return
        for n in self.sinks:
            arr = self.a[n]
            if n not in self.red:
                self.ctx.host_map(arr, D.R)
                self.ctx.host_unmap(arr)
            else:
                self.ctx.host_read(arr, C.addressof(self._scalar), 0, min(4, arr.nbytes))

    def run(self):
        if not self.streaming:  # resident: one batch call + the prepared sink reads
            key = (id(getattr(self, "L", None)), id(getattr(self, "it", None)))
            steps = getattr(self, "_steps", None)
            if steps is None or self._steps_key != key:
                self.launch_all()   # builds the batch for this key
                self.end_run()      # builds the prepared reads
                def status_of(fn):  # wrappers that raise on error -> return 0
                    def g():
                        fn()
                        return 0
                    return g
                b = self._batch
                call = b._fn if isinstance(b, D.Batch) else status_of(b)
                self._steps = [call] + [getattr(r, "call", None) or status_of(r) for r in self._reads]
                self._steps_key = key
                return
            for f in steps:
                if f():
                    self._fail(f)
            return
        self.begin_run()
        self.launch_all()
        self.end_run()

    def _fail(self, f):
        # redo the failing call through the raising wrapper for the message
        b = self._batch
        if isinstance(b, D.Batch) and f is b._fn:
            b()
        for r in self._reads:
            if getattr(r, "call", None) is f:
                r()
        raise RuntimeError("dagrt call failed")

    def launch_all(self):
        """The program's launches in order, issued by one dagrt_launch_batch
        call (identical to calling each prepared launch in turn).  Callables
        that are not prepared launches (e.g. tracing wrappers in tests) are
        called in turn."""
        # rebuilt when a launch list is replaced (set _batch = _steps = None after an
        # in-place edit of self.L / self.it)
        key = (id(getattr(self, "L", None)), id(getattr(self, "it", None)))
        if getattr(self, "_batch", None) is None or self._batch_key != key:
            seq = self.launch_sequence()
            self._batch_key = key
            self._batch = (self.ctx.batch(seq) if all(isinstance(L, D.Launch) for L in seq)
                           else (lambda: [L() for L in seq]))
        self._batch()

    def launch_sequence(self):
        """The prepared launches of one run, in program order."""
        return list(self.L)

    # ---------------------------------------------------------- baseline
    def graph(self):
        """Hand-written CUDA graph with manual dependencies (no inference)."""
        raise NotImplementedError

    def graph_io(self, g):
        """Stream mode: H2D nodes for inputs; returns {input name: node}."""
        if self.um:
            raise NotImplementedError("hand-written graphs take device or mirrored arrays, not UM")
        if self.mode != "stream":
            return {}
        return {n: g.copy(self.a[n], "h2d") for n in self.inputs}

    def graph_sinks(self, g, deps_of, only=None):
        """The graph's host reads of the sinks, so that it ends, like run(),
        with the host holding the outputs (same timed region for every
        schedule): whole arrays through the mirrors (stream) or
        one element per sink into pinned host memory (resident)."""
        if self.mode == "stream":
            for n in (only or self.sinks):
                g.copy(self.a[n], "d2h", nbytes=4 if n in self.red else None, deps=[deps_of[n]])
            return
        if self.record:
            return
        if getattr(self, "_graph_pin", None) is None:
            self._graph_pin = torch.zeros(16 * max(1, len(self.sinks)), dtype=torch.uint8,
                                          pin_memory=True)
        base = self._graph_pin.data_ptr()
        for n in (only or self.sinks):
            i = self.sinks.index(n)
            g.read(self.a[n], base + 16 * i, nbytes=min(4, self.a[n].nbytes), deps=[deps_of[n]])

    # ---------------------------------------------------------- bytes
    def kernel_bytes(self):
        """Algorithmic HBM bytes per vertex: {label: bytes}."""
        raise NotImplementedError

    def io_bytes(self):
        h2d = sum(self.t[n].numel() * self.t[n].element_size() for n in self.inputs)
        d2h = sum(4 if n in self.red else self.t[n].numel() * self.t[n].element_size()
                  for n in self.sinks)
        return (h2d, d2h) if self.streaming else (0, 4 * len(self.sinks))
