// libdagrt -- run-time DAG scheduler core (C++17), behind the C ABI of
// include/dagrt.h.  B200-native re-design of the scheduler of arXiv
// 2012.09646 (§IV); readings D1-D8 in DESIGN.md.
//
// Per launch (Fig. 5 steps 1-6, L630-639):
//   1 convert the invocation to a computational element (vertex)    L388-396
//   2-3 dependency inference from the per-array table:              L408-431, L490-491
//        read  -> last writer, if active                 (Fig. 3 A, C)
//        write -> active readers since the last writer, else the last
//                 writer if active                        (Fig. 3 B; D1)
//   4 stream: parent's stream if that parent is its tail, else the first
//     stream with no active vertex (FIFO), else a new stream  L570-582, L647-650
//   5 cudaStreamWaitEvent on parents living on other streams   L546-553
//     + prefetch of host-newer read args on the copy stream    L356-366, L662-664
//   6 launch, record the vertex event; return without blocking L564-569
// Host accesses (L505-530) wait on exactly the conflicting vertices' events
// and retire them and their DAG ancestors (L553-556; reading D4/D5).
//
// The scheduler keeps only the active frontier: per-array {last writer,
// readers since it}, per-vertex {active, stream, event, parents} -- parents
// are kept only to close retirement over ancestors and are dropped whenever
// the frontier empties.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/dagrt.h"
#include "builtin.h"

#include <nvtx3/nvToolsExt.h>

namespace dagrt {

// NVTX ranges (domain "dagrt") around launches, host accesses, barriers and
// graph-cache flushes: a profiler (nsys / ncu --nvtx) shows the scheduler's
// host timeline next to the GPU work.  Header-only NVTX3: without a tool
// attached every call is a null-pointer check.
static nvtxDomainHandle_t nvtx_domain() {
  static nvtxDomainHandle_t d = nvtxDomainCreateA("dagrt");
  return d;
}
struct NvtxRange {
  explicit NvtxRange(const char* name) {
    nvtxEventAttributes_t a{};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    nvtxDomainRangePushEx(nvtx_domain(), &a);
  }
  ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ------------------------------------------------------------ builtin registry
static std::vector<Builtin>& registry() {
  static std::vector<Builtin> r;
  return r;
}
static std::vector<std::pair<const void*, ResolveFn>>& resolvers() {
  static std::vector<std::pair<const void*, ResolveFn>> r;
  return r;
}
int register_builtins(const Builtin* t, int n) {
  for (int i = 0; i < n; ++i) registry().push_back(t[i]);
  return n;
}
int register_builtins_ext(const Builtin* t, int n, ResolveFn resolve) {
  for (int i = 0; i < n; ++i) {
    registry().push_back(t[i]);
    resolvers().push_back({t[i].fn, resolve});
  }
  return n;
}
ResolveFn builtin_resolver(const void* stub) {
  for (auto& r : resolvers())
    if (r.first == stub) return r.second;
  return nullptr;
}
int builtin_count() { return (int)registry().size(); }
const Builtin* builtin_at(int i) {
  return (i >= 0 && i < builtin_count()) ? &registry()[i] : nullptr;
}

// ------------------------------------------------------------ backends
// The CUDA runtime manager of Fig. 5 (L543-545, L590): the only place that
// talks to CUDA.  The recorder implements the same interface without a GPU.
struct Backend {
  virtual ~Backend() {}
  virtual cudaError_t stream_create(void** s) = 0;
  virtual cudaError_t stream_destroy(void* s) = 0;
  virtual cudaError_t event_create(void** e) = 0;
  virtual cudaError_t event_create_timing(void** e) = 0;
  virtual cudaError_t elapsed(float* ms, void* a, void* b) = 0;
  virtual cudaError_t event_destroy(void* e) = 0;
  virtual cudaError_t launch(const void* fn, dim3 g, dim3 b, void** args, size_t smem, void* s,
                             bool coop, int nargs) = 0;
  virtual cudaError_t record(void* e, void* s) = 0;
  virtual cudaError_t wait(void* s, void* e) = 0;
  virtual cudaError_t event_sync(void* e) = 0;
  virtual cudaError_t stream_sync(void* s) = 0;
  virtual cudaError_t copy_async(void* dst, const void* src, size_t n, cudaMemcpyKind k,
                                 void* s) = 0;
  virtual cudaError_t prefetch(void* p, size_t n, int dev, void* s) = 0;  // managed memory
  virtual bool real() const = 0;
};

struct CudaBackend final : Backend {
  cudaError_t stream_create(void** s) override {
    return cudaStreamCreateWithFlags(reinterpret_cast<cudaStream_t*>(s), cudaStreamNonBlocking);
  }
  cudaError_t stream_destroy(void* s) override { return cudaStreamDestroy((cudaStream_t)s); }
  cudaError_t event_create(void** e) override {
    return cudaEventCreateWithFlags(reinterpret_cast<cudaEvent_t*>(e), cudaEventDisableTiming);
  }
  cudaError_t event_create_timing(void** e) override {
    return cudaEventCreateWithFlags(reinterpret_cast<cudaEvent_t*>(e), cudaEventDefault);
  }
  cudaError_t elapsed(float* ms, void* a, void* b) override {
    return cudaEventElapsedTime(ms, (cudaEvent_t)a, (cudaEvent_t)b);
  }
  cudaError_t event_destroy(void* e) override { return cudaEventDestroy((cudaEvent_t)e); }
  // Kernels are enqueued through the driver's cuLaunchKernel on the kernel's
  // CUfunction (resolved once per host stub): measured 2.4 us per launch on
  // the B200 box's host vs 3.0 us for cudaLaunchKernel, which re-resolves the
  // stub on every call (tools/launch_cost.cu).  The entry point is fetched
  // from the runtime, so the library has no link-time dependency on libcuda.
  typedef int (*LaunchFn)(void* f, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by,
                          unsigned bz, unsigned smem, void* stream, void** params, void** extra);
  LaunchFn cu_launch = nullptr;
  bool cu_tried = false;
  std::vector<std::pair<const void*, void*>> funcs;  // host stub -> CUfunction
  typedef int (*FuncAttrFn)(void* f, int attrib, int value);
  FuncAttrFn cu_func_attr = nullptr;
  void* cufunc(const void* fn) {
    for (auto& p : funcs)
      if (p.first == fn) return p.second;
    void* f = nullptr;
    if (ResolveFn rs = builtin_resolver(fn)) {
      // a stub of another library's CUDA runtime (libdagrt_exp.so): its own
      // lookup, then the shared memory opt-in through the driver
      if (rs(fn, &f) != 0) f = nullptr;
      if (f) {
        if (!cu_func_attr) {
          void* p = nullptr;
          cudaDriverEntryPointQueryResult q;
          if (cudaGetDriverEntryPoint("cuFuncSetAttribute", &p, cudaEnableDefault, &q) == cudaSuccess &&
              q == cudaDriverEntryPointSuccess)
            cu_func_attr = (FuncAttrFn)p;
          cudaGetLastError();
        }
        for (int i = 0; i < builtin_count(); ++i)
          if (builtin_at(i)->fn == fn && builtin_at(i)->smem_max > 0 && cu_func_attr)
            cu_func_attr(f, 8 /* CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES */, builtin_at(i)->smem_max);
      }
    } else {
      cudaFunction_t cf = nullptr;
      if (cudaGetFuncBySymbol(&cf, fn) != cudaSuccess) {
        cudaGetLastError();
        cf = nullptr;
      }
      f = (void*)cf;
    }
    funcs.push_back({fn, f});
    return f;
  }
  cudaError_t launch(const void* fn, dim3 g, dim3 b, void** args, size_t smem, void* s,
                     bool coop, int) override {
    if (coop) {  // cooperative kernels are product kernels (launched by their own runtime's stub)
      if (builtin_resolver(fn)) return cudaErrorNotSupported;
      return cudaLaunchCooperativeKernel(fn, g, b, args, smem, (cudaStream_t)s);
    }
    if (!cu_tried) {
      cu_tried = true;
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuLaunchKernel", &p, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        cu_launch = (LaunchFn)p;
      else
        cudaGetLastError();
    }
    void* f = cu_launch ? cufunc(fn) : nullptr;
    if (!f && builtin_resolver(fn)) return cudaErrorInvalidDeviceFunction;  // not ours to launch by stub
    if (!f) return cudaLaunchKernel(fn, g, b, args, smem, (cudaStream_t)s);
    int r = cu_launch(f, g.x, g.y, g.z, b.x, b.y, b.z, (unsigned)smem, s, args, nullptr);
    // CUresult and cudaError_t share their numeric codes for launch failures
    // (invalid value 1, out of memory 2, invalid image 200, handle 400, 7xx)
    return (cudaError_t)r;
  }
  cudaError_t record(void* e, void* s) override {
    return cudaEventRecord((cudaEvent_t)e, (cudaStream_t)s);
  }
  cudaError_t wait(void* s, void* e) override {
    return cudaStreamWaitEvent((cudaStream_t)s, (cudaEvent_t)e, 0);
  }
  cudaError_t event_sync(void* e) override { return cudaEventSynchronize((cudaEvent_t)e); }
  cudaError_t stream_sync(void* s) override { return cudaStreamSynchronize((cudaStream_t)s); }
  cudaError_t copy_async(void* dst, const void* src, size_t n, cudaMemcpyKind k,
                         void* s) override {
    return cudaMemcpyAsync(dst, src, n, k, (cudaStream_t)s);
  }
  cudaError_t prefetch(void* p, size_t n, int dev, void* s) override {
    return cudaMemPrefetchAsync(p, n, dev, (cudaStream_t)s);
  }
  bool real() const override { return true; }
};

struct RecordBackend final : Backend {
  uintptr_t next = 0x1000;
  cudaError_t stream_create(void** s) override { *s = (void*)(next += 16); return cudaSuccess; }
  cudaError_t stream_destroy(void*) override { return cudaSuccess; }
  cudaError_t event_create(void** e) override { *e = (void*)(next += 16); return cudaSuccess; }
  cudaError_t event_create_timing(void** e) override { *e = (void*)(next += 16); return cudaSuccess; }
  cudaError_t elapsed(float* ms, void*, void*) override { *ms = 0.f; return cudaSuccess; }
  cudaError_t event_destroy(void*) override { return cudaSuccess; }
  cudaError_t launch(const void*, dim3, dim3, void**, size_t, void*, bool, int) override {
    return cudaSuccess;
  }
  cudaError_t record(void*, void*) override { return cudaSuccess; }
  cudaError_t wait(void*, void*) override { return cudaSuccess; }
  cudaError_t event_sync(void*) override { return cudaSuccess; }
  cudaError_t stream_sync(void*) override { return cudaSuccess; }
  cudaError_t copy_async(void*, const void*, size_t, cudaMemcpyKind, void*) override {
    return cudaSuccess;
  }
  cudaError_t prefetch(void*, size_t, int, void*) override { return cudaSuccess; }
  bool real() const override { return false; }
};

// ------------------------------------------------------------ graph cache
// Deferred submission + trace cache: while enabled, the stream operations
// the scheduler decides (launches, event records, cross-stream waits, copies)
// are buffered instead of issued.  At the next host synchronisation the
// buffered batch is keyed by its exact content; a batch seen for the second
// time is stream-captured into a CUDA graph (fork/join over every stream it
// uses, so the graph reproduces the scheduler's multi-stream schedule), and
// later identical batches replay that graph with one cudaGraphLaunch on a
// private in-order `origin` stream.  Dependencies are still inferred at run
// time for every launch; only the CUDA submission is cached.
//
// Events.  Every vertex event recorded inside a captured batch also gets an
// EXTERNAL event-record node of the graph (cudaEventRecordExternal) on a
// graph-owned event; after a replay the vertex's event is aliased to that
// node's event, so a host access or a later batch waits for exactly its
// producer, not for the whole graph.  Each stream's last operation in the
// graph likewise records a per-stream tail event: a stream synchronisation
// (the D2H of a host read) waits for that stream's part of the graph only.
//
// Ordering with work issued outside the graph (eagerly, on the scheduler's
// streams): a stream that got eager work since the last replay is forked
// into `origin` (event record + wait) before the next graph launch that uses
// it, and eager work on a stream whose tail ran inside a replayed graph
// first waits on that stream's tail event.  So same-stream order (which the
// scheduler relies on: a child on its parent's stream gets no event wait)
// holds across graph/eager boundaries in both directions.
struct DeferBackend final : Backend {
  enum : uint8_t { OP_LAUNCH, OP_RECORD, OP_WAIT, OP_COPY };
  struct Op {
    uint8_t kind;
    bool coop;
    int32_t nargs;
    void* s;
    void* e;
    const void* fn;
    dim3 g, b;
    size_t smem;
    uint64_t vals[17];
    void* dst;
    const void* src;
    size_t n;
    cudaMemcpyKind k;
  };
  struct Entry {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec = nullptr;
    std::vector<void*> rec_ev;                      // per OP_RECORD, in op order
    std::vector<std::pair<void*, void*>> tail_ev;   // (stream, tail event)
  };
  struct StreamState {
    void* s;
    bool dirty;      // eager work issued since the last fork into `origin`
    void* gtail;     // tail event of this stream in the last replay (or null)
    bool ordered;    // the stream already waits on gtail
  };
  Backend* in;
  bool enabled = false;
  void* origin = nullptr;
  std::vector<Op> ops;
  std::vector<uint64_t> key;
  std::vector<Entry> cache;                 // small, linear search by hash first
  std::vector<uint64_t> cache_hash;
  std::vector<uint64_t> seen;               // batch hashes seen once (eager)
  std::vector<uint64_t> nocap;              // batches whose capture failed (always eager)
  std::vector<std::pair<void*, void*>> alias;  // vertex event -> graph-owned event
  std::vector<StreamState> sstate;
  std::vector<void*> owned;                 // graph-owned events (destroyed with the cache)
  std::vector<void*> fork_evs;
  void* fork_ev = nullptr;
  uint64_t replays = 0, captures = 0, eager = 0;

  // Event-record nodes of a captured batch.  A vertex's event is needed
  // outside its batch only if later work or a host access waits on it (a
  // later batch, a host read of an earlier sink); every other record would
  // be an external event node that the graph executes for nothing (measured:
  // VEC 29.1 -> 27.7 us per DAG without them, tools/f1_lab.py).  So the
  // first, eager issue of a batch LEARNS which of its records escape (an
  // outside wait or sync on the event before it is recorded again), and the
  // capture gives only those their own event node; the others stand for
  // their stream's tail event in the graph -- later than the vertex on the
  // same stream, so a wait on it is still correct, only possibly longer.
  // DAGRT_F1_EVENTS=vertex (a node per vertex) / tail (none) for the labs.
  enum { EV_LEARN, EV_VERTEX, EV_TAIL } ev_mode = EV_LEARN;
  struct Pending { void* e; uint64_t h; uint32_t ord; };
  std::vector<Pending> pend;                                   // records of eager batches
  std::vector<std::pair<uint64_t, std::vector<uint32_t>>> esc;  // batch hash -> escaped record ordinals
  void note_escape(void* e) {
    for (size_t i = 0; i < pend.size(); ++i)
      if (pend[i].e == e) {
        std::vector<uint32_t>* v = nullptr;
        for (auto& x : esc)
          if (x.first == pend[i].h) v = &x.second;
        if (!v) {
          if (esc.size() >= 64) esc.erase(esc.begin());
          esc.push_back({pend[i].h, {}});
          v = &esc.back().second;
        }
        if (std::find(v->begin(), v->end(), pend[i].ord) == v->end()) v->push_back(pend[i].ord);
        pend[i] = pend.back();
        pend.pop_back();
        return;
      }
  }
  void forget_pending(void* e) {
    for (size_t i = 0; i < pend.size(); ++i)
      if (pend[i].e == e) {
        pend[i] = pend.back();
        pend.pop_back();
        return;
      }
  }
  bool escaped(uint64_t h, uint32_t ord) const {
    for (auto& x : esc)
      if (x.first == h) return std::find(x.second.begin(), x.second.end(), ord) != x.second.end();
    return false;
  }
  explicit DeferBackend(Backend* inner) : in(inner) {
    if (const char* t = getenv("DAGRT_F1_EVENTS")) {
      if (!strcmp(t, "vertex")) ev_mode = EV_VERTEX;
      if (!strcmp(t, "tail")) ev_mode = EV_TAIL;
    }
  }
  ~DeferBackend() override {
    for (auto& e : cache)
      if (e.exec) cudaGraphExecDestroy(e.exec);
    for (void* e : owned) in->event_destroy(e);
    for (void* e : fork_evs) in->event_destroy(e);
    if (fork_ev) in->event_destroy(fork_ev);
    if (origin) in->stream_destroy(origin);
    delete in;
  }
  bool active() const { return enabled; }
  bool graphs_used() const { return replays || captures; }

  void* resolve(void* e) const {
    for (auto& a : alias)
      if (a.first == e) return a.second;
    return e;
  }
  void unalias(void* e) {
    for (size_t i = 0; i < alias.size(); ++i)
      if (alias[i].first == e) {
        alias[i] = alias.back();
        alias.pop_back();
        return;
      }
  }
  StreamState* state(void* s) {
    for (auto& x : sstate)
      if (x.s == s) return &x;
    sstate.push_back(StreamState{s, true, nullptr, true});  // unknown: may hold eager work
    return &sstate.back();
  }
  // Before eager work on stream s: order it after s's part of the last graph.
  cudaError_t pre_eager(void* s) {
    if (!graphs_used() || !s) return cudaSuccess;
    StreamState* st = state(s);
    if (st->gtail && !st->ordered) {
      if (cudaError_t e = in->wait(s, st->gtail)) return e;
      st->ordered = true;
    }
    st->dirty = true;
    return cudaSuccess;
  }

  cudaError_t stream_create(void** s) override { return in->stream_create(s); }
  cudaError_t stream_destroy(void* s) override { return in->stream_destroy(s); }
  cudaError_t event_create(void** e) override { return in->event_create(e); }
  cudaError_t event_create_timing(void** e) override { return in->event_create_timing(e); }
  cudaError_t elapsed(float* ms, void* a, void* b) override { return in->elapsed(ms, a, b); }
  cudaError_t event_destroy(void* e) override { return in->event_destroy(e); }
  bool real() const override { return in->real(); }

  cudaError_t launch(const void* fn, dim3 g, dim3 b, void** args, size_t smem, void* s, bool coop,
                     int nargs) override {
    if (!enabled || nargs > 17) {
      if (cudaError_t e = flush()) return e;
      if (cudaError_t e = pre_eager(s)) return e;
      return in->launch(fn, g, b, args, smem, s, coop, nargs);
    }
    Op o{};
    o.kind = OP_LAUNCH;
    o.coop = coop;
    o.fn = fn;
    o.g = g;
    o.b = b;
    o.smem = smem;
    o.s = s;
    o.nargs = nargs;
    for (int i = 0; i < nargs; ++i) o.vals[i] = *reinterpret_cast<const uint64_t*>(args[i]);
    ops.push_back(o);
    return cudaSuccess;
  }
  cudaError_t record(void* e, void* s) override {
    unalias(e);
    forget_pending(e);
    if (!enabled) {
      if (cudaError_t r = pre_eager(s)) return r;
      return in->record(e, s);
    }
    Op o{};
    o.kind = OP_RECORD;
    o.e = e;
    o.s = s;
    ops.push_back(o);
    return cudaSuccess;
  }
  cudaError_t wait(void* s, void* e) override {
    note_escape(e);
    e = resolve(e);
    if (!enabled) {
      if (cudaError_t r = pre_eager(s)) return r;
      return in->wait(s, e);
    }
    Op o{};
    o.kind = OP_WAIT;
    o.e = e;
    o.s = s;
    ops.push_back(o);
    return cudaSuccess;
  }
  // A D2H copy into pinned memory (a host mirror or the context's bounce
  // buffer) joins the batch: the host access that issued it synchronises
  // right after, so the whole batch -- kernels, waits and the read-back --
  // replays as ONE graph launch, like a hand-written graph with a memcpy
  // node.  Other D2H copies (possibly pageable destinations) are issued
  // directly after the batch.
  bool d2h_pinned = false;
  cudaError_t copy_d2h_pinned(void* dst, const void* src, size_t n, void* s) {
    d2h_pinned = true;
    cudaError_t e = copy_async(dst, src, n, cudaMemcpyDeviceToHost, s);
    d2h_pinned = false;
    return e;
  }
  cudaError_t copy_async(void* dst, const void* src, size_t n, cudaMemcpyKind k, void* s) override {
    if (!enabled || (k == cudaMemcpyDeviceToHost && !d2h_pinned)) {
      if (cudaError_t e = flush()) return e;
      if (cudaError_t e = pre_eager(s)) return e;
      return in->copy_async(dst, src, n, k, s);
    }
    Op o{};
    o.kind = OP_COPY;
    o.dst = dst;
    o.src = src;
    o.n = n;
    o.k = k;
    o.s = s;
    ops.push_back(o);
    return cudaSuccess;
  }
  cudaError_t prefetch(void* p, size_t n, int dev, void* s) override {  // never deferred
    if (cudaError_t e = flush()) return e;
    if (cudaError_t e = pre_eager(s)) return e;
    return in->prefetch(p, n, dev, s);
  }
  cudaError_t event_sync(void* e) override {
    note_escape(e);
    if (cudaError_t r = flush()) return r;
    return in->event_sync(resolve(e));
  }
  cudaError_t stream_sync(void* s) override {
    if (cudaError_t r = flush()) return r;
    if (graphs_used()) {
      StreamState* st = state(s);
      // s's newest work is its part of a replayed graph: wait for that part only
      if (st->gtail && !st->ordered) return in->event_sync(st->gtail);
    }
    return in->stream_sync(s);
  }

  cudaError_t issue(const Op& o, bool capturing) {
    if (!capturing)
      if (cudaError_t e = pre_eager(o.s)) return e;
    switch (o.kind) {
      case OP_LAUNCH: {
        void* argv[17];
        for (int i = 0; i < o.nargs; ++i) argv[i] = const_cast<uint64_t*>(&o.vals[i]);
        return in->launch(o.fn, o.g, o.b, argv, o.smem, o.s, o.coop, o.nargs);
      }
      case OP_RECORD: return in->record(o.e, o.s);
      case OP_WAIT: return capturing ? cudaSuccess : in->wait(o.s, o.e);
      default: return in->copy_async(o.dst, o.src, o.n, o.k, o.s);
    }
  }

  // Batch key.  Event handles are canonicalised to their first-appearance
  // index: pooled events come back in varying order between identical runs,
  // and a captured graph does not depend on them (recorded-and-waited events
  // become graph edges, host-visible records are graph-owned events; external
  // waits are taken from the current batch when it is replayed).
  std::vector<void*> key_events;
  void build_key() {
    key.clear();
    key_events.clear();
    for (const Op& o : ops) {
      key.push_back(o.kind | (o.coop ? 0x100u : 0u));
      key.push_back((uint64_t)(uintptr_t)o.s);
      uint64_t ev = 0;
      if (o.e) {
        size_t i = 0;
        while (i < key_events.size() && key_events[i] != o.e) ++i;
        if (i == key_events.size()) key_events.push_back(o.e);
        ev = i + 1;
      }
      key.push_back(ev);
      if (o.kind == OP_LAUNCH) {
        key.push_back((uint64_t)(uintptr_t)o.fn);
        key.push_back(((uint64_t)o.g.x << 32) | o.g.y);
        key.push_back(((uint64_t)o.g.z << 32) | o.b.x);
        key.push_back(((uint64_t)o.b.y << 32) | o.b.z);
        key.push_back(o.smem);
        key.push_back((uint64_t)o.nargs);
        for (int i = 0; i < o.nargs; ++i) key.push_back(o.vals[i]);
      } else if (o.kind == OP_COPY) {
        key.push_back((uint64_t)(uintptr_t)o.dst);
        key.push_back((uint64_t)(uintptr_t)o.src);
        key.push_back(o.n);
        key.push_back((uint64_t)o.k);
      }
    }
  }
  static uint64_t hash(const std::vector<uint64_t>& k) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t v : k) {
      h ^= v;
      h *= 0x100000001b3ull;
      h ^= h >> 29;
    }
    return h;
  }

  // Waits on events that were not recorded earlier in this batch are
  // external dependencies: satisfied by making the origin stream wait on
  // them before the graph (a capture may not reference outside events).
  bool external_wait(size_t i) const {
    for (size_t j = 0; j < i; ++j)
      if (ops[j].kind == OP_RECORD && ops[j].e == ops[i].e) return false;
    return true;
  }
  bool is_owned(void* e) const { return std::find(owned.begin(), owned.end(), e) != owned.end(); }

  std::vector<void*> batch_streams() const {
    std::vector<void*> streams;
    for (const Op& o : ops)
      if (std::find(streams.begin(), streams.end(), o.s) == streams.end()) streams.push_back(o.s);
    return streams;
  }

  cudaError_t run_graph(Entry& en) {
    for (size_t i = 0; i < ops.size(); ++i)  // (events of earlier replays: origin is in order)
      if (ops[i].kind == OP_WAIT && external_wait(i) && !is_owned(ops[i].e))
        if (cudaError_t e = in->wait(origin, ops[i].e)) return e;
    // fork: streams with eager work since the last replay feed into origin
    size_t nf = 0;
    for (auto& te : en.tail_ev) {
      StreamState* st = state(te.first);
      if (!st->dirty) continue;
      if (nf == fork_evs.size()) {
        void* e;
        if (cudaError_t r = in->event_create(&e)) return r;
        fork_evs.push_back(e);
      }
      if (cudaError_t e = in->record(fork_evs[nf], te.first)) return e;
      if (cudaError_t e = in->wait(origin, fork_evs[nf])) return e;
      ++nf;
      st->dirty = false;
    }
    if (cudaError_t e = cudaGraphLaunch(en.exec, (cudaStream_t)origin)) return e;
    size_t r = 0;
    for (const Op& o : ops)
      if (o.kind == OP_RECORD) {
        unalias(o.e);
        alias.push_back({o.e, en.rec_ev[r++]});
      }
    for (auto& te : en.tail_ev) {
      StreamState* st = state(te.first);
      st->gtail = te.second;
      st->ordered = false;
    }
    return cudaSuccess;
  }

  cudaError_t owned_event(void** e) {
    if (cudaError_t r = in->event_create(e)) return r;
    owned.push_back(*e);
    return cudaSuccess;
  }

  cudaError_t capture(Entry* en, uint64_t h) {
    std::vector<void*> streams = batch_streams();
    if (!fork_ev)
      if (cudaError_t r = in->event_create(&fork_ev)) return r;
    std::vector<void*> join(streams.size());
    for (size_t i = 0; i < streams.size(); ++i) {
      if (cudaError_t r = owned_event(&join[i])) return r;
      en->tail_ev.push_back({streams[i], join[i]});
    }
    std::vector<bool> node;  // per record: its own external event node?
    for (const Op& o : ops)
      if (o.kind == OP_RECORD) {
        const uint32_t ord = (uint32_t)node.size();
        const bool own = ev_mode == EV_VERTEX || (ev_mode == EV_LEARN && escaped(h, ord));
        node.push_back(own);
        void* e = nullptr;
        if (!own) {  // the vertex's event stands for its stream's tail in the graph
          for (size_t i = 0; i < streams.size(); ++i)
            if (streams[i] == o.s) e = join[i];
        } else if (cudaError_t r = owned_event(&e)) {
          return r;
        }
        en->rec_ev.push_back(e);
      }
    cudaStream_t org = (cudaStream_t)origin;
    if (cudaError_t r = cudaStreamBeginCapture(org, cudaStreamCaptureModeRelaxed)) return r;
    cudaError_t err = in->record(fork_ev, origin);
    for (void* s : streams)
      if (!err) err = in->wait(s, fork_ev);
    size_t r = 0;
    for (size_t i = 0; i < ops.size() && !err; ++i) {
      if (ops[i].kind == OP_WAIT) {
        if (!external_wait(i)) err = in->wait(ops[i].s, ops[i].e);
      } else {
        err = issue(ops[i], true);
        if (!err && ops[i].kind == OP_RECORD && node[r++])
          err = cudaEventRecordWithFlags((cudaEvent_t)en->rec_ev[r - 1], (cudaStream_t)ops[i].s,
                                         cudaEventRecordExternal);
      }
    }
    for (size_t i = 0; i < streams.size() && !err; ++i) {
      err = cudaEventRecordWithFlags((cudaEvent_t)join[i], (cudaStream_t)streams[i], cudaEventRecordExternal);
      if (!err) err = in->record(fork_ev, streams[i]);  // join into origin (capture-internal)
      if (!err) err = in->wait(origin, fork_ev);
    }
    cudaGraph_t g = nullptr;
    cudaError_t end = cudaStreamEndCapture(org, &g);
    if (err) {
      if (g) cudaGraphDestroy(g);
      return err;
    }
    if (end) return end;
    cudaGraphExec_t exec = nullptr;
    cudaError_t ri = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    en->exec = exec;
    return ri;
  }

  cudaError_t flush() {
    if (ops.empty()) return cudaSuccess;
    NvtxRange nvtx_("dagrt_graph_cache_flush");
    if (!origin)
      if (cudaError_t e = in->stream_create(&origin)) return e;
    build_key();
    const uint64_t h = hash(key);
    cudaError_t err = cudaSuccess;
    bool done = false;
    for (size_t i = 0; i < cache.size() && !done; ++i)
      if (cache_hash[i] == h && cache[i].key == key) {
        err = run_graph(cache[i]);
        ++replays;
        done = true;
      }
    // Only batches with kernel launches are worth a graph: a batch of waits and
    // copies alone (the later host reads of a DAG whose kernels already went
    // out in an earlier graph) is issued eagerly on its own streams, where it
    // waits for exactly its producers -- a graph would queue it on `origin`
    // behind the whole earlier graph.
    bool has_launch = false;
    for (const Op& o : ops) has_launch = has_launch || o.kind == OP_LAUNCH;
    if (!done && has_launch && std::find(nocap.begin(), nocap.end(), h) == nocap.end() &&
        std::find(seen.begin(), seen.end(), h) != seen.end()) {
      Entry en;
      en.key = key;
      cudaError_t ce = capture(&en, h);
      if (!ce) {
        if (cache.size() >= 16) {
          cudaGraphExecDestroy(cache.front().exec);
          cache.erase(cache.begin());
          cache_hash.erase(cache_hash.begin());
        }
        cache.push_back(std::move(en));
        cache_hash.push_back(h);
        err = run_graph(cache.back());
        ++captures;
        done = true;
      } else {
        // not capturable (e.g. an operation the driver refuses to capture):
        // this batch is always issued eagerly from now on
        if (en.exec) cudaGraphExecDestroy(en.exec);
        cudaGetLastError();
        nocap.push_back(h);
      }
    }
    if (!done) {  // first sighting: issue eagerly, remember the batch and its records
      err = cudaSuccess;
      uint32_t ord = 0;
      for (const Op& o : ops) {
        if (!err) err = issue(o, false);
        if (o.kind == OP_RECORD) {
          forget_pending(o.e);
          if (pend.size() < 4096) pend.push_back(Pending{o.e, h, ord});
          ++ord;
        }
      }
      if (seen.size() >= 64) seen.erase(seen.begin());
      seen.push_back(h);
      ++eager;
    }
    ops.clear();
    return err;
  }

  // A stream wait issued right away (after flushing the batch): used to
  // order a D2H copy after its producers without blocking the host.
  cudaError_t wait_now(void* s, void* e) {
    note_escape(e);
    if (cudaError_t r = flush()) return r;
    if (cudaError_t r = pre_eager(s)) return r;
    return in->wait(s, resolve(e));
  }

  cudaError_t launch_now(const void* fn, dim3 g, dim3 b, void** args, size_t smem, void* s, bool coop) {
    if (cudaError_t e = flush()) return e;
    if (cudaError_t e = pre_eager(s)) return e;
    return in->launch(fn, g, b, args, smem, s, coop, 0);
  }
};

// ------------------------------------------------------------ context state
enum : uint8_t { P_I32 = 0, P_I64 = 1, P_CONST = 2, P_INOUT = 3, P_OUT = 4, P_F32 = 5, P_F64 = 6 };
inline bool is_ptr(uint8_t k) { return k >= P_CONST && k <= P_OUT; }
enum : uint8_t { COH_DEVICE = 0, COH_HOST = 1, COH_BOTH = 2 };  // which copy is newest

constexpr int kMaxArgs = 16;

struct KernelRec {
  std::string name;
  const void* fn;
  PrelaunchFn pre = nullptr;  // built-in pre-launch hook (extra leading kernel argument)
  ValidateFn validate = nullptr;  // built-in launch contract
  int32_t nparams;
  uint8_t kind[kMaxArgs];
  bool coop;
  bool prof = false;
  bool lib = false;  // pseudo-kernel of library-call vertices (dagrt_launch_library)
  std::vector<dagrt_launch_config> cands;  // history-driven launch configuration (f3)
  int32_t trials = 0;
};

// Per (kernel, scalar-argument key) launch history of an auto-configured kernel.
struct TuneRec {
  uint32_t kernel;
  uint64_t key;
  std::vector<std::vector<float>> ms;  // samples per candidate
  int32_t next = 0;                    // round-robin cursor while exploring
  int32_t chosen = -1;
};
struct TunePending {
  size_t rec;
  int32_t cand;
  void* ev0;
  void* ev1;
};

struct ProfRec {
  uint32_t kernel;
  void* ev0;
  void* ev1;
};

struct TimeRec {
  int32_t kind, stream;
  int64_t vertex, id;
  uint64_t bytes;
  void* ev0;
  void* ev1;
};

struct ArrayRec {
  char* dev = nullptr;
  char* host = nullptr;
  size_t bytes = 0;
  uint32_t gen = 0;
  bool live = false;
  bool mapped = false;
  bool managed = false;             // unified memory: dev == host, no copies (dagrt_array_register_managed)
  bool host_touched = false;        // managed: the host accessed it since the last device prefetch
  int64_t last_writer = -1;         // GLOBAL vertex id of the last kernel writer, -1 = none/host
  std::vector<int64_t> readers;     // global ids of the readers since the last writer (pruned lazily)
  uint8_t coh = COH_DEVICE;
  bool h2d_pending = false;         // an H2D prefetch whose consumer is still active
  void* h2d_ev = nullptr;
  int64_t h2d_consumer = -1;        // global vertex id
  int32_t h2d_stream = -1;          // stream of the consumer (already ordered after the copy)
};

struct VertexRec {
  uint8_t active;
  uint8_t kind;   // 0 kernel, 1 host
  int32_t stream;
  void* ev;
  uint32_t pbeg, pcnt;  // parents in parent_pool
};

struct StreamRec {
  void* s;
  int64_t tail;    // last enqueued vertex
  int32_t nactive; // active vertices on this stream
};

struct GraphRec {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaGraphNode_t> nodes;
};

}  // namespace dagrt

using namespace dagrt;

struct dagrt_graph_s {
  GraphRec r;
};

struct dagrt_ctx_s {
  dagrt_config cfg{};
  int device = 0;
  DeferBackend* be = nullptr;  // wraps the CUDA / record backend (graph cache)
  std::string err;
  bool sticky = false;

  std::vector<KernelRec> kernels;
  std::vector<ArrayRec> arrays;       // index 0 unused (handle 0 invalid)
  // Vertex table of the current EPOCH: local index i is global vertex id
  // vid_base + i.  When the active frontier empties (every vertex retired by
  // host syncs), the table and the parent links are dropped and vid_base
  // advances (recycle()): the scheduler's state stays bounded by the frontier
  // instead of growing with every launch.  Arrays and streams keep global
  // ids, which simply become inactive.
  std::vector<VertexRec> vertices;
  int64_t vid_base = 0;
  std::vector<uint32_t> parent_pool;
  std::vector<StreamRec> streams;
  std::vector<void*> event_pool;      // free events
  std::vector<void*> all_events;
  int64_t n_active = 0;
  void* copy_stream = nullptr;        // in-order H2D side stream
  void* d2h_stream = nullptr;         // in-order D2H side stream
  void* graph_stream = nullptr;
  void* serial_stream = nullptr;
  void* bounce = nullptr;              // pinned staging for small D2H reads into caller memory
  void* mapped = nullptr;              // mapped pinned memory for small host reads (+ flag word)
  void* mapped_dev = nullptr;          // its device address
  uint32_t read_seq = 0;
  std::vector<dagrt_graph_s*> graphs;
  std::vector<ProfRec> prof;           // timed launches awaiting collection
  std::vector<TuneRec> tune;           // launch-configuration history (f3)
  std::vector<TunePending> tune_pending;
  int64_t tune_last = -1;              // TuneRec of the last auto launch
  int64_t tune_req_rec = -1;           // the launch being enqueued is an exploration sample of
  int32_t tune_req_cand = -1;          //   (TuneRec, candidate): do_launch brackets it with events
  bool timeline = false;
  std::vector<TimeRec> tl;             // timeline records awaiting export
  std::vector<void*> tev_pool;         // free timing events
  std::vector<void*> all_tev;

  // introspection
  std::vector<dagrt_vertex_info> rec_v;
  std::vector<dagrt_edge_info> rec_e;
  std::vector<dagrt_trace_op> trace;
  dagrt_stats_t st{};

  // scratch reused across launches (no per-launch heap traffic)
  std::vector<std::pair<uint32_t, uint32_t>> scratch_edges;  // (parent vid, array idx)
  std::vector<uint32_t> scratch_parents;
  std::vector<uint32_t> stack;
};

namespace {

dagrt_status fail(dagrt_ctx c, dagrt_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  c->err = buf;
  return s;
}

dagrt_status cuda_fail(dagrt_ctx c, cudaError_t e, const char* what) {
  c->sticky = true;
  return fail(c, DAGRT_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define CK(call, what)                                   \
  do {                                                   \
    cudaError_t e__ = (call);                            \
    if (e__ != cudaSuccess) return cuda_fail(c, e__, what); \
  } while (0)

#define GUARD(c)                                                   \
  do {                                                             \
    if (!(c)) return DAGRT_EINVAL;                                 \
    if ((c)->sticky) return DAGRT_ECUDA;                           \
  } while (0)

inline void trace_op(dagrt_ctx c, int32_t op, int32_t stream, int64_t a, int64_t b, uint64_t bytes) {
  if (c->cfg.record_dag) c->trace.push_back(dagrt_trace_op{op, stream, a, b, bytes});
}

ArrayRec* get_array(dagrt_ctx c, dagrt_array h) {
  uint32_t idx = (uint32_t)(h & 0xffffffffu);
  uint32_t gen = (uint32_t)(h >> 32);
  if (idx == 0 || idx >= c->arrays.size()) return nullptr;
  ArrayRec* a = &c->arrays[idx];
  if (!a->live || a->gen != gen) return nullptr;
  return a;
}

inline uint32_t array_index(dagrt_ctx c, const ArrayRec* a) { return (uint32_t)(a - c->arrays.data()); }
inline dagrt_array array_handle(dagrt_ctx c, const ArrayRec* a) {
  return ((uint64_t)a->gen << 32) | array_index(c, a);
}

inline bool is_active(dagrt_ctx c, int64_t gid) {
  const int64_t v = gid - c->vid_base;
  return gid >= 0 && v >= 0 && (size_t)v < c->vertices.size() && c->vertices[v].active;
}
inline uint32_t local_of(dagrt_ctx c, int64_t gid) { return (uint32_t)(gid - c->vid_base); }

dagrt_status get_event(dagrt_ctx c, void** ev) {
  if (!c->event_pool.empty()) {
    *ev = c->event_pool.back();
    c->event_pool.pop_back();
    return DAGRT_OK;
  }
  CK(c->be->event_create(ev), "cudaEventCreate");
  c->all_events.push_back(*ev);
  c->st.events_created++;
  return DAGRT_OK;
}

dagrt_status get_timing_event(dagrt_ctx c, void** ev) {
  if (!c->tev_pool.empty()) {
    *ev = c->tev_pool.back();
    c->tev_pool.pop_back();
    return DAGRT_OK;
  }
  CK(c->be->event_create_timing(ev), "cudaEventCreate timing");
  c->all_tev.push_back(*ev);
  return DAGRT_OK;
}

float median_of(std::vector<float> v) {
  std::sort(v.begin(), v.end());
  return v.empty() ? -1.f : v[v.size() / 2];
}

// Collect the finished timings of exploring auto launches (non-blocking:
// cudaEventQuery), and decide a configuration once every candidate has its
// trials.
void tune_collect(dagrt_ctx c) {
  if (c->tune_pending.empty()) return;
  std::vector<TunePending> keep;
  for (const TunePending& t : c->tune_pending) {
    float ms = 0.f;
    bool done = true;
    if (c->be->real()) {
      cudaError_t q = cudaEventQuery((cudaEvent_t)t.ev1);
      if (q == cudaErrorNotReady) {
        keep.push_back(t);
        continue;
      }
      cudaGetLastError();
      done = q == cudaSuccess && cudaEventElapsedTime(&ms, (cudaEvent_t)t.ev0, (cudaEvent_t)t.ev1) == cudaSuccess;
      cudaGetLastError();
    }
    if (done) c->tune[t.rec].ms[t.cand].push_back(ms);
    c->tev_pool.push_back(t.ev0);
    c->tev_pool.push_back(t.ev1);
  }
  c->tune_pending.swap(keep);
  for (TuneRec& r : c->tune) {
    if (r.chosen >= 0) continue;
    const KernelRec& k = c->kernels[r.kernel];
    bool all = true;
    for (const auto& v : r.ms) all = all && (int32_t)v.size() >= k.trials;
    if (!all) continue;
    int32_t best = 0;
    for (size_t i = 1; i < r.ms.size(); ++i)
      if (median_of(r.ms[i]) < median_of(r.ms[best])) best = (int32_t)i;
    r.chosen = best;
  }
}

// The one place kernels are enqueued; optionally bracketed by timing events
// on the launching stream (dagrt_profile_enable).
// Timeline bracket (dagrt_timeline_enable): opens before an item on stream s.
dagrt_status tl_begin(dagrt_ctx c, void* s, void** e0) {
  *e0 = nullptr;
  if (!c->timeline) return DAGRT_OK;
  if (dagrt_status st = get_timing_event(c, e0)) return st;
  CK(c->be->record(*e0, s), "cudaEventRecord timeline");
  return DAGRT_OK;
}
dagrt_status tl_end(dagrt_ctx c, void* s, void* e0, int32_t kind, int32_t sidx, int64_t vertex,
                    int64_t id, uint64_t bytes) {
  if (!c->timeline || !e0) return DAGRT_OK;
  void* e1;
  if (dagrt_status st = get_timing_event(c, &e1)) return st;
  CK(c->be->record(e1, s), "cudaEventRecord timeline");
  c->tl.push_back(TimeRec{kind, sidx, vertex, id, bytes, e0, e1});
  return DAGRT_OK;
}

// The one place kernels are enqueued; optionally bracketed by timing events
// on the launching stream (dagrt_profile_enable / dagrt_timeline_enable).
dagrt_status do_launch(dagrt_ctx c, const KernelRec* k, uint32_t kh, dim3 g, dim3 b, void** argv,
                       uint32_t smem, void* s, int32_t sidx = -1, int64_t vertex = -1) {
  void *e0 = nullptr, *e1 = nullptr, *t0 = nullptr;
  if (k->prof) {
    if (dagrt_status st = get_timing_event(c, &e0)) return st;
    if (dagrt_status st = get_timing_event(c, &e1)) return st;
    CK(c->be->record(e0, s), "cudaEventRecord profile");
  }
  void *u0 = nullptr, *u1 = nullptr;
  if (c->tune_req_rec >= 0) {  // exploration sample of an auto-configured launch (f3)
    if (dagrt_status st = get_timing_event(c, &u0)) return st;
    if (dagrt_status st = get_timing_event(c, &u1)) return st;
    CK(c->be->record(u0, s), "cudaEventRecord autotune");
  }
  if (dagrt_status st = tl_begin(c, s, &t0)) return st;
  CK(c->be->launch(k->fn, g, b, argv, smem, s, k->coop, k->nparams + (k->pre ? 1 : 0)), "cudaLaunchKernel");
  if (dagrt_status st = tl_end(c, s, t0, 0, sidx, vertex, kh, 0)) return st;
  if (u0) {
    CK(c->be->record(u1, s), "cudaEventRecord autotune");
    c->tune_pending.push_back(TunePending{(size_t)c->tune_req_rec, c->tune_req_cand, u0, u1});
    c->tune_req_rec = -1;
  }
  if (k->prof) {
    CK(c->be->record(e1, s), "cudaEventRecord profile");
    c->prof.push_back(ProfRec{kh, e0, e1});
  }
  return DAGRT_OK;
}

inline uint64_t now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Retire vertex v and all its active ancestors (D4/D5: a host sync on v
// proves v and everything v waited on have completed).
void retire(dagrt_ctx c, uint32_t v) {
  auto& stk = c->stack;
  stk.clear();
  stk.push_back(v);
  while (!stk.empty()) {
    uint32_t k = stk.back();
    stk.pop_back();
    VertexRec& vr = c->vertices[k];
    if (!vr.active) continue;
    vr.active = 0;
    c->n_active--;
    if (vr.stream >= 0) c->streams[vr.stream].nactive--;
    if (vr.ev) {
      c->event_pool.push_back(vr.ev);
      vr.ev = nullptr;
    }
    for (uint32_t i = 0; i < vr.pcnt; ++i) {
      uint32_t p = c->parent_pool[vr.pbeg + i];
      if (c->vertices[p].active) stk.push_back(p);
    }
  }
  if (c->n_active == 0) c->parent_pool.clear();  // frontier empty: parent links no longer needed
}

void retire_all(dagrt_ctx c) {
  for (size_t v = 0; v < c->vertices.size() && c->n_active > 0; ++v)
    if (c->vertices[v].active) retire(c, (uint32_t)v);
}

// New epoch once the frontier is empty (see dagrt_ctx_s::vertices).
void recycle(dagrt_ctx c) {
  if (c->n_active != 0 || c->vertices.empty()) return;
  c->vid_base += (int64_t)c->vertices.size();
  c->vertices.clear();
  c->parent_pool.clear();
}

// Drop readers that are no longer active (amortised: when the list grows)
void prune_readers(dagrt_ctx c, ArrayRec* a) {
  auto& rd = a->readers;
  size_t w = 0;
  for (size_t i = 0; i < rd.size(); ++i)
    if (is_active(c, rd[i])) rd[w++] = rd[i];
  rd.resize(w);
}

// Dependency inference for one access (array a, write?) against the active
// frontier; appends (parent, array) pairs to scratch_edges.
void infer(dagrt_ctx c, ArrayRec* a, bool write) {
  uint32_t ai = array_index(c, a);
  if (!write) {
    if (is_active(c, a->last_writer)) c->scratch_edges.push_back({local_of(c, a->last_writer), ai});
    return;
  }
  prune_readers(c, a);
  auto& rd = a->readers;
  if (!rd.empty()) {
    for (int64_t r : rd) c->scratch_edges.push_back({local_of(c, r), ai});
  } else if (is_active(c, a->last_writer)) {
    c->scratch_edges.push_back({local_of(c, a->last_writer), ai});
  }
}

// Sorted unique parent list from scratch_edges; records edge rows.
void collect_parents(dagrt_ctx c, uint32_t child) {
  auto& e = c->scratch_edges;
  std::sort(e.begin(), e.end());
  e.erase(std::unique(e.begin(), e.end()), e.end());
  auto& ps = c->scratch_parents;
  ps.clear();
  for (auto& pr : e) {
    if (ps.empty() || ps.back() != pr.first) ps.push_back(pr.first);
    if (c->cfg.record_dag)
      c->rec_e.push_back(dagrt_edge_info{(uint32_t)(c->vid_base + pr.first), (uint32_t)(c->vid_base + child),
                                         array_handle(c, &c->arrays[pr.second])});
  }
  c->st.edges += ps.size();
}

dagrt_status new_stream(dagrt_ctx c, int32_t* out) {
  void* s = nullptr;
  CK(c->be->stream_create(&s), "cudaStreamCreate");
  c->streams.push_back(StreamRec{s, -1, 0});
  c->st.streams++;
  *out = (int32_t)c->streams.size() - 1;
  return DAGRT_OK;
}

// Stream manager (L570-582, L647-654; stream oracle in SURVEY §8(c1)).
dagrt_status pick_stream(dagrt_ctx c, int32_t* out) {
  if (c->cfg.policy == DAGRT_PARALLEL_SINGLE_STREAM && !c->scratch_parents.empty() &&
      c->vertices[c->scratch_parents[0]].stream >= 0) {
    // "schedule all children on a single stream" (L650-654): the first parent's
    *out = c->vertices[c->scratch_parents[0]].stream;
    return DAGRT_OK;
  }
  for (uint32_t p : c->scratch_parents) {
    int32_t s = c->vertices[p].stream;
    if (s >= 0 && c->streams[s].tail == c->vid_base + (int64_t)p) { *out = s; return DAGRT_OK; }
  }
  for (size_t s = 0; s < c->streams.size(); ++s)
    if (c->streams[s].nactive == 0) { *out = (int32_t)s; return DAGRT_OK; }
  if (c->cfg.max_streams <= 0 || (int)c->streams.size() < c->cfg.max_streams)
    return new_stream(c, out);
  // capped: the first parent's stream, else the least loaded stream
  if (!c->scratch_parents.empty() && c->vertices[c->scratch_parents[0]].stream >= 0) {
    *out = c->vertices[c->scratch_parents[0]].stream;
    return DAGRT_OK;
  }
  int32_t best = 0;
  for (size_t s = 1; s < c->streams.size(); ++s)
    if (c->streams[s].nactive < c->streams[best].nactive) best = (int32_t)s;
  *out = best;
  return DAGRT_OK;
}

// Host blocks on exactly the conflicting vertices (L553-555), then retires them.
// With `order` (a D2H stream) the wait is not a separate host round trip: the
// stream is made to wait on the parents' events and the caller's copy + one
// stream synchronisation on it block the host until parents and copy are
// done -- the same ordering, one host wake-up instead of two.
dagrt_status host_sync_parents(dagrt_ctx c, ArrayRec* a, bool write, void* order = nullptr) {
  c->scratch_edges.clear();
  infer(c, a, write);
  if (c->scratch_edges.empty()) {
    if (write) { a->readers.clear(); a->last_writer = -1; }
    return DAGRT_OK;  // not modelled as a DAG element (L512-516)
  }
  uint32_t vid = (uint32_t)c->vertices.size();
  collect_parents(c, vid);
  c->vertices.push_back(VertexRec{0, 1, -1, nullptr, 0, 0});
  c->st.vertices++;
  c->st.host_vertices++;
  if (c->cfg.record_dag)
    c->rec_v.push_back(dagrt_vertex_info{(uint32_t)(c->vid_base + vid), 1, 0, -1, array_handle(c, a)});
  for (uint32_t p : c->scratch_parents) {
    trace_op(c, DAGRT_OP_EVENT_SYNC, -1, c->vid_base + p, 0, 0);
    // (with the graph cache on, the wait joins the pending batch with the copy)
    if (order && c->be->active()) CK(c->be->wait(order, c->vertices[p].ev), "cudaStreamWaitEvent D2H");
    else if (order) CK(c->be->wait_now(order, c->vertices[p].ev), "cudaStreamWaitEvent D2H");
    else CK(c->be->event_sync(c->vertices[p].ev), "cudaEventSynchronize");
    c->st.host_syncs++;
  }
  for (uint32_t p : c->scratch_parents) retire(c, p);
  if (write) { a->readers.clear(); a->last_writer = -1; }
  recycle(c);
  tune_collect(c);
  return DAGRT_OK;
}

constexpr size_t kBounceBytes = 64 << 10;
constexpr size_t kMappedReadBytes = 4096;

// Small read through mapped pinned memory: a one-CTA kernel on the D2H stream
// (ordered after the producers by the waits host_sync_parents put there)
// copies the bytes and publishes a sequence number; the host spins on it,
// polling the stream every 256 spins so a failed or finished stream is seen.
dagrt_status d2h_mapped(dagrt_ctx c, ArrayRec* a, size_t off, size_t n, void* dst) {
  if (!c->mapped) {
    CK(cudaHostAlloc(&c->mapped, kMappedReadBytes + 64, cudaHostAllocMapped), "cudaHostAlloc mapped");
    CK(cudaHostGetDevicePointer(&c->mapped_dev, c->mapped, 0), "cudaHostGetDevicePointer");
  }
  volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>((char*)c->mapped + kMappedReadBytes);
  uint32_t seq = ++c->read_seq;
  if (seq == 0) seq = c->read_seq = 1;
  const char* src = a->dev + off;
  char* ddst = (char*)c->mapped_dev;
  uint32_t nn = (uint32_t)n;
  uint32_t* dflag = reinterpret_cast<uint32_t*>(ddst + kMappedReadBytes);
  void* argv[] = {&src, &ddst, &nn, &dflag, &seq};
  void* t0;
  if (dagrt_status st_ = tl_begin(c, c->d2h_stream, &t0)) return st_;
  CK(c->be->launch(read_mapped_kernel(), dim3(1), dim3(256), argv, 0, c->d2h_stream, false, 5),
     "cudaLaunchKernel mapped read");
  if (dagrt_status st_ = tl_end(c, c->d2h_stream, t0, 2, -5, -1, array_index(c, a), n)) return st_;
  for (uint32_t it = 1; *flag != seq; ++it) {
    if ((it & 255) == 0) {
      cudaError_t q = cudaStreamQuery((cudaStream_t)c->d2h_stream);
      if (q == cudaSuccess) {
        if (*flag != seq) return fail(c, DAGRT_ECUDA, "mapped host read: stream idle, flag not set");
        break;
      }
      if (q != cudaErrorNotReady) CK(q, "cudaStreamQuery D2H");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  c->st.host_syncs++;
  memcpy(dst, c->mapped, n);
  return DAGRT_OK;
}

dagrt_status d2h(dagrt_ctx c, ArrayRec* a, size_t off, size_t n, void* dst) {
  if (n == 0) return DAGRT_OK;
  if (a->managed) {  // the host reads unified memory in place
    a->host_touched = true;
    if (c->cfg.prefetch) {  // move the range to the host first (DMA) instead of CPU page faults
      c->st.um_prefetch_bytes += n;
      CK(c->be->prefetch(a->dev + off, n, cudaCpuDeviceId, c->d2h_stream), "cudaMemPrefetchAsync to host");
      CK(c->be->stream_sync(c->d2h_stream), "cudaStreamSynchronize D2H");
      c->st.host_syncs++;
    }
    if (c->be->real() && dst != a->dev + off) memcpy(dst, a->dev + off, n);
    return DAGRT_OK;
  }
  trace_op(c, DAGRT_OP_D2H, -1, array_index(c, a), (int64_t)off, n);
  c->st.d2h_bytes += n;
  c->st.d2h_copies++;
  if (!c->be->real()) return DAGRT_OK;
  // Small reads use the mapped-memory kernel only when none of this
  // context's vertices is still active: then the one-CTA kernel starts at
  // once.  With kernels in flight it would queue behind their CTAs for an SM
  // slot (B&S: reads of the first sinks while nine pricing kernels fill the
  // GPU measured 0.54 vs 0.45 ms per DAG), so the copy engine does the read.
  // (With the graph cache on, reads stay memcpy nodes of the replayed batch.)
  if (n <= kMappedReadBytes && !c->be->active() && c->n_active == 0) return d2h_mapped(c, a, off, n, dst);
  // small reads into caller (possibly pageable) memory go through a pinned
  // bounce buffer: a pageable D2H is staged by the driver and much slower
  const bool bounce = n <= kBounceBytes && !(a->host && (char*)dst >= a->host &&
                                             (char*)dst < a->host + a->bytes);
  if (bounce && !c->bounce) CK(cudaMallocHost(&c->bounce, kBounceBytes), "cudaMallocHost bounce");
  void* t0;
  if (dagrt_status st_ = tl_begin(c, c->d2h_stream, &t0)) return st_;
  const bool pinned = bounce || (a->host && (char*)dst >= a->host && (char*)dst < a->host + a->bytes);
  if (pinned) {
    CK(c->be->copy_d2h_pinned(bounce ? c->bounce : dst, a->dev + off, n, c->d2h_stream), "cudaMemcpyAsync D2H");
  } else {
    CK(c->be->copy_async(dst, a->dev + off, n, cudaMemcpyDeviceToHost, c->d2h_stream), "cudaMemcpyAsync D2H");
  }
  if (dagrt_status st_ = tl_end(c, c->d2h_stream, t0, 2, -5, -1, array_index(c, a), n)) return st_;
  CK(c->be->stream_sync(c->d2h_stream), "cudaStreamSynchronize D2H");
  c->st.host_syncs++;
  if (bounce) memcpy(dst, c->bounce, n);
  return DAGRT_OK;
}

dagrt_status ensure_streams(dagrt_ctx c) {
  if (!c->copy_stream) {
    CK(c->be->stream_create(&c->copy_stream), "cudaStreamCreate copy");
    CK(c->be->stream_create(&c->d2h_stream), "cudaStreamCreate d2h");
    CK(c->be->stream_create(&c->graph_stream), "cudaStreamCreate graph");
    CK(c->be->stream_create(&c->serial_stream), "cudaStreamCreate serial");
  }
  return DAGRT_OK;
}

dagrt_status parse_signature(const char* sig, KernelRec* k) {
  k->nparams = 0;
  std::string s(sig ? sig : "");
  size_t pos = 0;
  if (s.find_first_not_of(" \t") == std::string::npos) return DAGRT_OK;
  while (pos <= s.size()) {
    size_t comma = s.find(',', pos);
    std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
    // normalise whitespace
    std::string norm;
    bool sp = false;
    for (char ch : tok) {
      if (ch == ' ' || ch == '\t') { sp = !norm.empty(); continue; }
      if (sp) { norm += ' '; sp = false; }
      norm += ch;
    }
    uint8_t kind;
    if (norm == "const ptr" || norm == "in ptr" || norm == "const pointer" || norm == "in pointer")
      kind = P_CONST;
    else if (norm == "ptr" || norm == "inout ptr" || norm == "pointer" || norm == "inout pointer")
      kind = P_INOUT;
    else if (norm == "out ptr" || norm == "out pointer")
      kind = P_OUT;
    else if (norm == "sint32" || norm == "uint32" || norm == "int")
      kind = P_I32;
    else if (norm == "float")
      kind = P_F32;
    else if (norm == "sint64" || norm == "uint64")
      kind = P_I64;
    else if (norm == "double")
      kind = P_F64;
    else
      return DAGRT_ESIG;
    if (k->nparams >= kMaxArgs) return DAGRT_ESIG;
    k->kind[k->nparams++] = kind;
    if (comma == std::string::npos) break;
    pos = comma + 1;
  }
  return DAGRT_OK;
}

// Launch configuration limits of the device (any kernel), then the
// built-in's own contract.  Both fail with DAGRT_EINVAL (not sticky): nothing
// was enqueued.
dagrt_status check_launch(dagrt_ctx c, const KernelRec& k, dim3 g, dim3 b, uint32_t smem, const uint64_t* vals,
                          ArrayRec* const* arrs, int nargs) {
  const uint64_t nt = (uint64_t)b.x * b.y * b.z;
  if (nt == 0 || nt > 1024) return fail(c, DAGRT_EINVAL, "kernel %s: block of %llu threads", k.name.c_str(),
                                        (unsigned long long)nt);
  if (g.x == 0 || g.y == 0 || g.z == 0 || g.y > 65535 || g.z > 65535)
    return fail(c, DAGRT_EINVAL, "kernel %s: grid (%u, %u, %u)", k.name.c_str(), g.x, g.y, g.z);
  if (smem > 227u * 1024u) return fail(c, DAGRT_EINVAL, "kernel %s: %u bytes of shared memory", k.name.c_str(), smem);
  if (!k.validate) return DAGRT_OK;
  uint64_t bytes[kMaxArgs];
  for (int i = 0; i < nargs; ++i) bytes[i] = arrs[i] ? arrs[i]->bytes : 0;
  LaunchCheck L{vals, bytes, nargs, {g.x, g.y, g.z}, {b.x, b.y, b.z}, smem, c->be->real()};
  if (const char* why = k.validate(L)) return fail(c, DAGRT_EINVAL, "kernel %s: %s", k.name.c_str(), why);
  return DAGRT_OK;
}

// Resolve args to the kernel parameter buffer; validates kinds.
dagrt_status marshal(dagrt_ctx c, const KernelRec& k, const dagrt_arg* args, int32_t nargs,
                     uint64_t* vals, void** argv, ArrayRec** arrs, dim3 g, dim3 b, uint32_t smem) {
  if (nargs != k.nparams)
    return fail(c, DAGRT_ESIG, "kernel %s: %d args given, signature has %d", k.name.c_str(), nargs,
                k.nparams);
  if (nargs > 0 && !args) return fail(c, DAGRT_EINVAL, "null args");
  for (int i = 0; i < nargs; ++i) {
    uint8_t kd = k.kind[i];
    if (is_ptr(kd)) {
      ArrayRec* a = get_array(c, args[i].array);
      if (!a) return fail(c, DAGRT_ENOTFOUND, "kernel %s arg %d: not a live array handle", k.name.c_str(), i);
      if (a->mapped) return fail(c, DAGRT_ESTATE, "kernel %s arg %d: array is host-mapped", k.name.c_str(), i);
      arrs[i] = a;
      vals[i] = (uint64_t)(uintptr_t)a->dev;
    } else {
      arrs[i] = nullptr;
      vals[i] = (uint64_t)args[i].i64;
      if (kd == P_I32 || kd == P_F32) vals[i] &= 0xffffffffull;
    }
    argv[i] = &vals[i];
  }
  if (dagrt_status st = check_launch(c, k, g, b, smem, vals, arrs, nargs)) return st;
  if (k.pre) {  // the hook's value becomes the kernel's first parameter (after validation)
    void* extra = nullptr;  // (no device work on the record backend: no hook)
    if (c->be->real())
      if (int e = k.pre(vals, nargs, &extra)) return cuda_fail(c, (cudaError_t)e, "pre-launch hook");
    for (int i = nargs; i > 0; --i) vals[i] = vals[i - 1];
    vals[0] = (uint64_t)(uintptr_t)extra;
    for (int i = 0; i <= nargs; ++i) argv[i] = &vals[i];
  }
  return DAGRT_OK;
}

dagrt_status lookup_kernel(dagrt_ctx c, dagrt_kernel k, KernelRec** out) {
  if (k >= c->kernels.size()) return fail(c, DAGRT_ENOTFOUND, "kernel handle %u", k);
  *out = &c->kernels[k];
  return DAGRT_OK;
}

}  // namespace

// =================================================================== C ABI
// A context's record of built-in b (handles 0..n-1 at creation; built-ins a
// library registers later -- libdagrt_exp.so -- are appended on lookup).
static dagrt_status add_builtin(dagrt_ctx c, const Builtin* b) {
  KernelRec k;
  k.name = b->name;
  k.fn = b->fn;
  k.coop = (b->flags & KF_COOPERATIVE) != 0;
  k.pre = b->prelaunch;
  k.validate = b->validate;
  if (b->smem_max > 0 && c->be->real() && b->fn && !builtin_resolver(b->fn))
    cudaFuncSetAttribute(b->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, b->smem_max);
  if (parse_signature(b->signature, &k) != DAGRT_OK) return DAGRT_ESIG;
  c->kernels.push_back(k);
  return DAGRT_OK;
}

extern "C" {

dagrt_status dagrt_create(int device, const dagrt_config* cfg, dagrt_ctx* out) {
  if (!out) return DAGRT_EINVAL;
  *out = nullptr;
  dagrt_ctx c = new (std::nothrow) dagrt_ctx_s();
  if (!c) return DAGRT_ENOMEM;
  if (cfg) c->cfg = *cfg;
  else c->cfg = dagrt_config{DAGRT_PARALLEL_ASYNC, 1, 0, 0, DAGRT_BACKEND_CUDA, 0};
  c->device = device;
  if (c->cfg.backend == DAGRT_BACKEND_RECORD) {
    c->be = new DeferBackend(new RecordBackend());
  } else {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
      delete c;
      return DAGRT_ECUDA;
    }
    c->be = new DeferBackend(new CudaBackend());
    c->be->enabled = c->cfg.graph_cache != 0 && c->cfg.policy != DAGRT_SERIAL_SYNC;
  }
  c->arrays.resize(1);
  // built-in kernels are pre-registered (handles 0..n-1)
  for (int i = 0; i < builtin_count(); ++i) {
    if (add_builtin(c, builtin_at(i)) != DAGRT_OK) {
      delete c->be;
      delete c;
      return DAGRT_ESIG;
    }
  }
  if (ensure_streams(c) != DAGRT_OK) {
    delete c->be;
    delete c;
    return DAGRT_ECUDA;
  }
  c->scratch_edges.reserve(64);
  c->scratch_parents.reserve(64);
  *out = c;
  return DAGRT_OK;
}

dagrt_status dagrt_destroy(dagrt_ctx c) {
  if (!c) return DAGRT_OK;
  c->be->flush();
  if (c->be->real()) {
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
  }
  for (auto* g : c->graphs) {
    if (g->r.exec) cudaGraphExecDestroy(g->r.exec);
    if (g->r.g) cudaGraphDestroy(g->r.g);
    delete g;
  }
  for (void* e : c->all_events) c->be->event_destroy(e);
  for (void* e : c->all_tev) c->be->event_destroy(e);
  for (auto& s : c->streams) c->be->stream_destroy(s.s);
  for (void* s : {c->copy_stream, c->d2h_stream, c->graph_stream, c->serial_stream})
    if (s) c->be->stream_destroy(s);
  for (auto& a : c->arrays)
    if (a.h2d_ev) c->be->event_destroy(a.h2d_ev);
  if (c->bounce) cudaFreeHost(c->bounce);
  if (c->mapped) cudaFreeHost(c->mapped);
  delete c->be;
  delete c;
  return DAGRT_OK;
}

const char* dagrt_last_error(dagrt_ctx c) { return c ? c->err.c_str() : "null context"; }

dagrt_status dagrt_array_register(dagrt_ctx c, void* dev, void* host, size_t bytes,
                                  dagrt_array* out) {
  GUARD(c);
  if (!out) return fail(c, DAGRT_EINVAL, "null out");
  if (!dev && bytes) return fail(c, DAGRT_EINVAL, "null device pointer");
  if (bytes) {
    uintptr_t b0 = (uintptr_t)dev, b1 = b0 + bytes;
    for (size_t i = 1; i < c->arrays.size(); ++i) {
      const ArrayRec& a = c->arrays[i];
      if (!a.live || !a.bytes) continue;
      uintptr_t a0 = (uintptr_t)a.dev, a1 = a0 + a.bytes;
      if (b0 < a1 && a0 < b1)
        return fail(c, DAGRT_EALIAS, "device range [%p,+%zu) overlaps array %zu", dev, bytes, i);
    }
  }
  // reuse a dead slot if any
  size_t idx = 0;
  for (size_t i = 1; i < c->arrays.size(); ++i)
    if (!c->arrays[i].live) { idx = i; break; }
  if (!idx) {
    c->arrays.emplace_back();
    idx = c->arrays.size() - 1;
  }
  ArrayRec& a = c->arrays[idx];
  uint32_t gen = a.gen + 1;
  void* keep_ev = a.h2d_ev;
  a = ArrayRec();
  a.h2d_ev = keep_ev;
  a.gen = gen;
  a.dev = (char*)dev;
  a.host = (char*)host;
  a.bytes = bytes;
  a.live = true;
  *out = array_handle(c, &a);
  return DAGRT_OK;
}

dagrt_status dagrt_array_register_managed(dagrt_ctx c, void* ptr, size_t bytes, dagrt_array* out) {
  GUARD(c);
  if (!out) return fail(c, DAGRT_EINVAL, "null out");
  if (c->be->real() && ptr) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess || at.type != cudaMemoryTypeManaged) {
      cudaGetLastError();
      return fail(c, DAGRT_EINVAL, "%p is not managed memory (cudaMallocManaged)", ptr);
    }
  }
  if (dagrt_status s = dagrt_array_register(c, ptr, ptr, bytes, out)) return s;
  ArrayRec* a = get_array(c, *out);
  a->managed = true;
  a->host_touched = true;  // where its pages are is unknown
  a->coh = COH_BOTH;
  if (c->be->enabled) {  // prefetches are issued eagerly: no graph cache in UM mode
    CK(c->be->flush(), "graph cache flush");
    c->be->enabled = false;
  }
  return DAGRT_OK;
}

dagrt_status dagrt_managed_alloc(size_t bytes, void** p) {
  if (!p) return DAGRT_EINVAL;
  return cudaMallocManaged(p, bytes ? bytes : 1, cudaMemAttachGlobal) == cudaSuccess ? DAGRT_OK : DAGRT_ECUDA;
}
dagrt_status dagrt_managed_free(void* p) { return cudaFree(p) == cudaSuccess ? DAGRT_OK : DAGRT_ECUDA; }
dagrt_status dagrt_managed_to_host(void* p, size_t bytes) {
  if (!p) return DAGRT_EINVAL;
  if (cudaMemPrefetchAsync(p, bytes, cudaCpuDeviceId, 0) != cudaSuccess) return DAGRT_ECUDA;
  return cudaStreamSynchronize(0) == cudaSuccess ? DAGRT_OK : DAGRT_ECUDA;
}

dagrt_status dagrt_array_unregister(dagrt_ctx c, dagrt_array h) {
  GUARD(c);
  ArrayRec* a = get_array(c, h);
  if (!a) return fail(c, DAGRT_ENOTFOUND, "array handle");
  // wait for in-flight users: the last writer, active readers, a pending copy
  if (is_active(c, a->last_writer)) {
    CK(c->be->event_sync(c->vertices[local_of(c, a->last_writer)].ev), "cudaEventSynchronize");
    c->st.host_syncs++;
  }
  for (int64_t r : a->readers)
    if (is_active(c, r)) {
      CK(c->be->event_sync(c->vertices[local_of(c, r)].ev), "cudaEventSynchronize");
      c->st.host_syncs++;
    }
  if (a->h2d_pending) {
    CK(c->be->event_sync(a->h2d_ev), "cudaEventSynchronize");
    a->h2d_pending = false;
  }
  a->live = false;
  a->readers.clear();
  a->readers.shrink_to_fit();
  return DAGRT_OK;
}

dagrt_status dagrt_array_device_ptr(dagrt_ctx c, dagrt_array h, void** dev) {
  GUARD(c);
  ArrayRec* a = get_array(c, h);
  if (!a || !dev) return fail(c, DAGRT_ENOTFOUND, "array handle");
  *dev = a->dev;
  return DAGRT_OK;
}

dagrt_status dagrt_kernel_register(dagrt_ctx c, const void* fn, const char* name,
                                   const char* signature, dagrt_kernel* out) {
  GUARD(c);
  if (!name || !out) return fail(c, DAGRT_EINVAL, "null name/out");
  if (!fn && c->be->real()) return fail(c, DAGRT_EINVAL, "null kernel function");
  KernelRec k;
  k.name = name;
  k.fn = fn;
  k.coop = false;
  if (parse_signature(signature, &k) != DAGRT_OK)
    return fail(c, DAGRT_ESIG, "bad signature '%s'", signature ? signature : "(null)");
  c->kernels.push_back(k);
  *out = (dagrt_kernel)(c->kernels.size() - 1);
  return DAGRT_OK;
}

dagrt_status dagrt_kernel_lookup(dagrt_ctx c, const char* name, dagrt_kernel* out) {
  GUARD(c);
  if (!name || !out) return fail(c, DAGRT_EINVAL, "null name/out");
  // user registrations shadow built-ins: search from the end
  for (size_t i = c->kernels.size(); i-- > 0;)
    if (c->kernels[i].name == name) {
      *out = (dagrt_kernel)i;
      return DAGRT_OK;
    }
  for (int i = 0; i < builtin_count(); ++i)  // registered after the context was created
    if (std::strcmp(builtin_at(i)->name, name) == 0) {
      if (dagrt_status s = add_builtin(c, builtin_at(i))) return fail(c, s, "bad signature of '%s'", name);
      *out = (dagrt_kernel)(c->kernels.size() - 1);
      return DAGRT_OK;
    }
  return fail(c, DAGRT_ENOTFOUND, "no kernel named '%s'", name);
}

dagrt_status dagrt_kernel_signature(dagrt_ctx c, dagrt_kernel k, int32_t* kinds, int32_t* n) {
  GUARD(c);
  KernelRec* kr;
  if (dagrt_status s = lookup_kernel(c, k, &kr)) return s;
  if (!n) return fail(c, DAGRT_EINVAL, "null n");
  int32_t cap = *n;
  *n = kr->nparams;
  if (!kinds) return DAGRT_OK;
  if (cap < kr->nparams) return fail(c, DAGRT_EINVAL, "capacity");
  for (int i = 0; i < kr->nparams; ++i) kinds[i] = kr->kind[i];
  return DAGRT_OK;
}

const char* dagrt_kernel_name(dagrt_ctx c, dagrt_kernel k) {
  if (!c || k >= c->kernels.size()) return nullptr;
  return c->kernels[k].name.c_str();
}

int32_t dagrt_builtin_count(void) { return builtin_count(); }
const char* dagrt_builtin_name(int32_t i) {
  const Builtin* b = builtin_at(i);
  return b ? b->name : nullptr;
}
const char* dagrt_builtin_signature(int32_t i) {
  const Builtin* b = builtin_at(i);
  return b ? b->signature : nullptr;
}

}  // extern "C"

namespace {
// One computational element (L388-396): a kernel (lib == nullptr) or a
// library call that enqueues its own GPU work on the stream the scheduler
// picks (L516-519).  arrs / kinds: the arguments and their access modes.
dagrt_status launch_vertex(dagrt_ctx c, KernelRec* k, dagrt_kernel kh, dagrt_dim3 grid, dagrt_dim3 block,
                           uint32_t smem, void** argv, ArrayRec* const* arrs, const uint8_t* kinds, int32_t nargs,
                           dagrt_library_fn lib, void* user, std::chrono::steady_clock::time_point t0);
}  // namespace

extern "C" {

dagrt_status dagrt_launch(dagrt_ctx c, dagrt_kernel kh, dagrt_dim3 grid, dagrt_dim3 block,
                          uint32_t smem, const dagrt_arg* args, int32_t nargs) {
  GUARD(c);
  auto t0 = std::chrono::steady_clock::now();
  KernelRec* k;
  if (dagrt_status s = lookup_kernel(c, kh, &k)) return s;
  if (k->lib) return fail(c, DAGRT_EINVAL, "%s is a library-call name, not a kernel", k->name.c_str());
  if (grid.x == 0 && grid.y == 0 && grid.z == 0) {  // auto configuration (f3)
    if (k->cands.empty()) return fail(c, DAGRT_EINVAL, "kernel %s: auto grid without dagrt_kernel_autotune", k->name.c_str());
    if (nargs != k->nparams || (nargs > 0 && !args)) return fail(c, DAGRT_ESIG, "kernel %s: argument count", k->name.c_str());
    uint64_t key = 0xcbf29ce484222325ull ^ kh;
    for (int i = 0; i < nargs; ++i)
      if (!is_ptr(k->kind[i])) key = (key ^ (uint64_t)args[i].i64) * 0x100000001b3ull;
    size_t r = 0;
    while (r < c->tune.size() && !(c->tune[r].kernel == kh && c->tune[r].key == key)) ++r;
    if (r == c->tune.size()) {
      TuneRec tr;
      tr.kernel = kh;
      tr.key = key;
      tr.ms.resize(k->cands.size());
      c->tune.push_back(tr);
    }
    tune_collect(c);
    TuneRec& tr = c->tune[r];
    c->tune_last = (int64_t)r;
    int32_t pick = tr.chosen;
    if (pick < 0) {
      if (c->be->active()) {  // graph cache on: no exploration (timing events are not replayable)
        pick = 0;
      } else {
        // next candidate still short of samples (launched or pending)
        const int32_t nc = (int32_t)k->cands.size();
        for (int32_t tries = 0; tries < nc; ++tries) {
          const int32_t cand = (tr.next + tries) % nc;
          int32_t have = (int32_t)tr.ms[cand].size();
          for (const TunePending& tp : c->tune_pending) have += tp.rec == r && tp.cand == cand;
          if (have < k->trials) { pick = cand; break; }
        }
        if (pick < 0) pick = tr.next % nc;  // all sampled, awaiting collection
        tr.next = (pick + 1) % nc;
        c->tune_req_rec = (int64_t)r;
        c->tune_req_cand = pick;
      }
    }
    const dagrt_launch_config& cf = k->cands[pick];
    grid = cf.grid;
    block = cf.block;
    smem = cf.smem;
  }
  uint64_t vals[kMaxArgs + 1];
  void* argv[kMaxArgs + 1];
  ArrayRec* arrs[kMaxArgs];
  if (dagrt_status s = marshal(c, *k, args, nargs, vals, argv, arrs, dim3(grid.x, grid.y, grid.z),
                               dim3(block.x, block.y, block.z), smem))
    return s;
  const dagrt_status st = launch_vertex(c, k, kh, grid, block, smem, argv, arrs, k->kind, nargs, nullptr, nullptr, t0);
  c->tune_req_rec = -1;
  return st;
}

dagrt_status dagrt_kernel_autotune(dagrt_ctx c, dagrt_kernel kh, const dagrt_launch_config* cands, int32_t n,
                                   int32_t trials) {
  GUARD(c);
  KernelRec* k;
  if (dagrt_status s = lookup_kernel(c, kh, &k)) return s;
  if (n < 1 || n > 16 || !cands || trials < 1) return fail(c, DAGRT_EINVAL, "autotune: 1..16 candidates, trials >= 1");
  k->cands.assign(cands, cands + n);
  k->trials = trials;
  for (size_t i = 0; i < c->tune.size(); ++i)  // a new candidate list restarts this kernel's history
    if (c->tune[i].kernel == kh) {
      c->tune[i].ms.assign((size_t)n, {});
      c->tune[i].chosen = -1;
      c->tune[i].next = 0;
    }
  std::vector<TunePending> keep;
  for (const TunePending& t : c->tune_pending)
    if (c->tune[t.rec].kernel != kh) keep.push_back(t);
  c->tune_pending.swap(keep);
  return DAGRT_OK;
}

dagrt_status dagrt_autotune_state(dagrt_ctx c, dagrt_kernel kh, int32_t* chosen, double* ms, int32_t* n) {
  GUARD(c);
  if (!chosen || !n) return fail(c, DAGRT_EINVAL, "null out");
  tune_collect(c);
  int64_t r = -1;
  for (size_t i = 0; i < c->tune.size(); ++i)
    if (c->tune[i].kernel == kh && (r < 0 || (int64_t)i == c->tune_last)) r = (int64_t)i;
  if (r < 0) return fail(c, DAGRT_ENOTFOUND, "no auto launch of kernel %u yet", kh);
  const TuneRec& tr = c->tune[r];
  *chosen = tr.chosen;
  const int32_t cap = *n;
  *n = (int32_t)tr.ms.size();
  if (ms) {
    if (cap < *n) return fail(c, DAGRT_EINVAL, "capacity");
    for (int32_t i = 0; i < *n; ++i) ms[i] = tr.ms[i].empty() ? -1.0 : (double)median_of(tr.ms[i]);
  }
  return DAGRT_OK;
}

dagrt_status dagrt_launch_library(dagrt_ctx c, dagrt_library_fn fn, void* user, const char* name,
                                  const dagrt_array* arrays, const int32_t* modes, int32_t n) {
  GUARD(c);
  auto t0 = std::chrono::steady_clock::now();
  if (!fn || !name || n < 0 || n > kMaxArgs || (n > 0 && (!arrays || !modes)))
    return fail(c, DAGRT_EINVAL, "library call: null function / name or bad array list");
  ArrayRec* arrs[kMaxArgs];
  uint8_t kinds[kMaxArgs];
  for (int i = 0; i < n; ++i) {
    ArrayRec* a = get_array(c, arrays[i]);
    if (!a) return fail(c, DAGRT_ENOTFOUND, "library call %s arg %d: not a live array handle", name, i);
    if (a->mapped) return fail(c, DAGRT_ESTATE, "library call %s arg %d: array is host-mapped", name, i);
    if (modes[i] < DAGRT_R || modes[i] > DAGRT_RW) return fail(c, DAGRT_EINVAL, "library call %s: mode %d", name, modes[i]);
    arrs[i] = a;
    kinds[i] = modes[i] == DAGRT_R ? P_CONST : (modes[i] == DAGRT_W ? P_OUT : P_INOUT);
  }
  // a pseudo-kernel per call name (for the DAG export and statistics)
  dagrt_kernel kh = 0;
  bool found = false;
  for (size_t i = c->kernels.size(); i-- > 0;)
    if (c->kernels[i].fn == nullptr && c->kernels[i].name == name && c->kernels[i].lib) {
      kh = (dagrt_kernel)i;
      found = true;
      break;
    }
  if (!found) {
    KernelRec kr;
    kr.name = name;
    kr.fn = nullptr;
    kr.nparams = 0;
    kr.coop = false;
    kr.lib = true;
    c->kernels.push_back(kr);
    kh = (dagrt_kernel)(c->kernels.size() - 1);
  }
  return launch_vertex(c, &c->kernels[kh], kh, dagrt_dim3{1, 1, 1}, dagrt_dim3{1, 1, 1}, 0, nullptr, arrs, kinds, n,
                       fn, user, t0);
}

}  // extern "C"

namespace {
// Enqueue the vertex's GPU work on stream s: the kernel, or the library call.
dagrt_status enqueue(dagrt_ctx c, KernelRec* k, dagrt_kernel kh, dim3 g, dim3 b, void** argv, uint32_t smem, void* s,
                     int32_t sidx, int64_t gvid, dagrt_library_fn lib, void* user) {
  if (!lib) return do_launch(c, k, kh, g, b, argv, smem, s, sidx, gvid);
  if (!c->be->real()) return DAGRT_OK;  // the recorder does no device work
  // a host callback cannot be deferred into a captured batch
  CK(c->be->flush(), "graph cache flush");
  CK(c->be->pre_eager(s), "graph cache ordering");
  if (int32_t r = lib(s, user)) return fail(c, DAGRT_EINVAL, "library call %s returned %d", k->name.c_str(), r);
  return DAGRT_OK;
}

// Does argument a of a vertex need a transfer before the vertex runs?  A
// mirrored array: it is read (need) and the host copy is newer.  A managed
// array (UM mode, D13): with prefetch on, whenever the host touched it since
// the last prefetch -- reads AND writes, since pages left on the host would
// otherwise be faulted in by the kernel; with prefetch off never (the faults
// are the mode), counting the host-newer bytes the kernel will fault in.
static bool transfer_needed(dagrt_ctx c, ArrayRec* a, bool need) {
  if (!a->bytes || !a->host) return false;
  if (!a->managed) return need && a->coh == COH_HOST;
  if (c->cfg.prefetch) return a->host_touched;
  if (need && a->coh == COH_HOST) {
    c->st.um_fault_bytes += a->bytes;
    a->coh = COH_BOTH;
  }
  return false;
}

dagrt_status launch_vertex(dagrt_ctx c, KernelRec* k, dagrt_kernel kh, dagrt_dim3 grid, dagrt_dim3 block,
                           uint32_t smem, void** argv, ArrayRec* const* arrs, const uint8_t* kinds, int32_t nargs,
                           dagrt_library_fn lib, void* user, std::chrono::steady_clock::time_point t0) {
  NvtxRange nvtx_(k->name.c_str());

  // merged access per distinct array (D3): write if any use writes,
  // needs data if any use reads (const / inout)
  ArrayRec* acc[kMaxArgs];
  bool wr[kMaxArgs], need[kMaxArgs];
  int nacc = 0;
  for (int i = 0; i < nargs; ++i) {
    if (!arrs[i]) continue;
    int j = 0;
    while (j < nacc && acc[j] != arrs[i]) ++j;
    if (j == nacc) { acc[nacc] = arrs[i]; wr[nacc] = false; need[nacc] = false; ++nacc; }
    uint8_t kd = kinds[i];
    if (kd != P_CONST) wr[j] = true;
    if (kd != P_OUT) need[j] = true;
  }
  dim3 g(grid.x, grid.y, grid.z), b(block.x, block.y, block.z);
  uint32_t vid = (uint32_t)c->vertices.size();  // local index in this epoch
  const int64_t gvid = c->vid_base + vid;        // global vertex id (exports, tables)
  c->st.launches++;
  c->st.vertices++;

  if (c->cfg.policy == DAGRT_SERIAL_SYNC) {
    // L560-569 / L908-909: program order on one stream, no dependency
    // computation, host waits after every copy and kernel.
    void* s = c->serial_stream;
    for (int j = 0; j < nacc; ++j) {
      ArrayRec* a = acc[j];
      if (transfer_needed(c, a, need[j])) {
        trace_op(c, DAGRT_OP_H2D, -3, array_index(c, a), 0, a->bytes);
        c->st.h2d_bytes += a->bytes;
        c->st.h2d_copies++;
        if (a->managed) c->st.um_prefetch_bytes += a->bytes;
        if (c->be->real()) {
          void* t0;
          if (dagrt_status st_ = tl_begin(c, s, &t0)) return st_;
          if (a->managed)
            CK(c->be->prefetch(a->dev, a->bytes, c->device, s), "cudaMemPrefetchAsync");
          else
            CK(c->be->copy_async(a->dev, a->host, a->bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync H2D");
          if (dagrt_status st_ = tl_end(c, s, t0, 1, -3, gvid, array_index(c, a), a->bytes)) return st_;
          CK(c->be->stream_sync(s), "cudaStreamSynchronize");
          c->st.host_syncs++;
        }
        if (need[j]) a->coh = COH_BOTH;
        a->host_touched = false;
      }
    }
    trace_op(c, DAGRT_OP_LAUNCH, -3, gvid, kh, 0);
    if (dagrt_status st_ = enqueue(c, k, kh, g, b, argv, smem, s, -3, gvid, lib, user)) return st_;
    CK(c->be->stream_sync(s), "cudaStreamSynchronize");
    c->st.host_syncs++;
    c->vertices.push_back(VertexRec{0, 0, -1, nullptr, 0, 0});
    recycle(c);  // nothing is ever active under the serial policy
    if (c->cfg.record_dag) c->rec_v.push_back(dagrt_vertex_info{(uint32_t)gvid, 0, kh, -1, 0});
    for (int j = 0; j < nacc; ++j)
      if (wr[j] && acc[j]->host) acc[j]->coh = COH_DEVICE;
    c->st.sched_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                          std::chrono::steady_clock::now() - t0).count();
    return DAGRT_OK;
  }

  // (2-3) dependencies from the dependency sets of active computations
  c->scratch_edges.clear();
  for (int j = 0; j < nacc; ++j) infer(c, acc[j], wr[j]);
  collect_parents(c, vid);

  // (4) stream
  int32_t sid;
  if (dagrt_status s = pick_stream(c, &sid)) return s;
  void* s = c->streams[sid].s;

  // (5) events: wait on parents running on other streams (one wait each)
  const uint64_t tw0 = now_ns();
  for (uint32_t p : c->scratch_parents) {
    const VertexRec& pv = c->vertices[p];
    if (pv.stream != sid) {
      trace_op(c, DAGRT_OP_WAIT, sid, c->vid_base + p, 0, 0);
      CK(c->be->wait(s, pv.ev), "cudaStreamWaitEvent");
      c->st.cross_stream_waits++;
    }
  }
  // transfers: prefetch host-newer inputs; order after pending prefetches
  for (int j = 0; j < nacc; ++j) {
    ArrayRec* a = acc[j];
    if (a->h2d_pending && !is_active(c, a->h2d_consumer)) a->h2d_pending = false;
    if (transfer_needed(c, a, need[j])) {
      void* cs = c->cfg.prefetch ? c->copy_stream : s;
      trace_op(c, DAGRT_OP_H2D, c->cfg.prefetch ? -2 : sid, array_index(c, a), 0, a->bytes);
      c->st.h2d_bytes += a->bytes;
      c->st.h2d_copies++;
      if (a->managed) c->st.um_prefetch_bytes += a->bytes;
      void* t0;
      if (dagrt_status st_ = tl_begin(c, cs, &t0)) return st_;
      if (a->managed)
        CK(c->be->prefetch(a->dev, a->bytes, c->device, cs), "cudaMemPrefetchAsync");
      else
        CK(c->be->copy_async(a->dev, a->host, a->bytes, cudaMemcpyHostToDevice, cs), "cudaMemcpyAsync H2D");
      if (dagrt_status st_ = tl_end(c, cs, t0, 1, c->cfg.prefetch ? -2 : sid, gvid, array_index(c, a),
                                    a->bytes))
        return st_;
      if (need[j]) a->coh = COH_BOTH;
      a->host_touched = false;
      // the copy's event orders every later reader on another stream after
      // it (with prefetch off the copy runs on this consumer's own stream, so
      // only those other readers wait)
      if (!a->h2d_ev) CK(c->be->event_create(&a->h2d_ev), "cudaEventCreate");
      CK(c->be->record(a->h2d_ev, cs), "cudaEventRecord copy");
      if (c->cfg.prefetch) {
        trace_op(c, DAGRT_OP_WAIT_COPY, sid, array_index(c, a), 0, 0);
        CK(c->be->wait(s, a->h2d_ev), "cudaStreamWaitEvent copy");
        c->st.copy_waits++;
      }
      a->h2d_pending = true;
      a->h2d_consumer = gvid;
      a->h2d_stream = sid;  // ordered after the copy in both modes
    } else if (a->h2d_pending && a->h2d_stream != sid) {
      trace_op(c, DAGRT_OP_WAIT_COPY, sid, array_index(c, a), 0, 0);
      CK(c->be->wait(s, a->h2d_ev), "cudaStreamWaitEvent copy");
      c->st.copy_waits++;
    }
  }

  // (6) launch + event
  void* ev;
  if (dagrt_status st = get_event(c, &ev)) return st;
  const uint64_t tl0 = now_ns();
  c->st.wait_ns += tl0 - tw0;
  trace_op(c, DAGRT_OP_LAUNCH, sid, gvid, kh, 0);
  if (dagrt_status st_ = enqueue(c, k, kh, g, b, argv, smem, s, sid, gvid, lib, user)) return st_;
  const uint64_t tr0 = now_ns();
  c->st.launch_ns += tr0 - tl0;
  trace_op(c, DAGRT_OP_RECORD, sid, gvid, 0, 0);
  CK(c->be->record(ev, s), "cudaEventRecord");
  c->st.record_ns += now_ns() - tr0;

  // bookkeeping: vertex, frontier, dependency sets
  uint32_t pbeg = (uint32_t)c->parent_pool.size();
  c->parent_pool.insert(c->parent_pool.end(), c->scratch_parents.begin(), c->scratch_parents.end());
  c->vertices.push_back(VertexRec{1, 0, sid, ev, pbeg, (uint32_t)c->scratch_parents.size()});
  c->n_active++;
  c->streams[sid].tail = gvid;
  c->streams[sid].nactive++;
  if (c->cfg.record_dag) c->rec_v.push_back(dagrt_vertex_info{(uint32_t)gvid, 0, kh, sid, 0});
  for (int j = 0; j < nacc; ++j) {
    ArrayRec* a = acc[j];
    if (wr[j]) {
      a->last_writer = gvid;
      a->readers.clear();
      if (a->host) a->coh = COH_DEVICE;
    } else {
      if (a->readers.size() >= 32) prune_readers(c, a);  // never-written arrays stay bounded
      a->readers.push_back(gvid);
    }
  }
  c->st.sched_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now() - t0).count();
  return DAGRT_OK;
}

}  // namespace

extern "C" {

dagrt_status dagrt_launch_prepared(dagrt_ctx c, const dagrt_launch_desc* d) {
  if (!d) return c ? fail(c, DAGRT_EINVAL, "null launch descriptor") : DAGRT_EINVAL;
  return dagrt_launch(c, d->kernel, d->grid, d->block, d->smem, d->args, d->nargs);
}

dagrt_status dagrt_launch_batch(dagrt_ctx c, const dagrt_launch_desc* d, int32_t n) {
  if (n < 0 || (n > 0 && !d)) return c ? fail(c, DAGRT_EINVAL, "bad launch batch") : DAGRT_EINVAL;
  for (int32_t i = 0; i < n; ++i)
    if (dagrt_status s = dagrt_launch(c, d[i].kernel, d[i].grid, d[i].block, d[i].smem, d[i].args, d[i].nargs))
      return s;
  return DAGRT_OK;
}

dagrt_status dagrt_host_read(dagrt_ctx c, dagrt_array h, size_t off, size_t bytes, void* dst) {
  NvtxRange nvtx_("dagrt_host_read");
  GUARD(c);
  ArrayRec* a = get_array(c, h);
  if (!a) return fail(c, DAGRT_ENOTFOUND, "array handle");
  if (off > a->bytes || bytes > a->bytes - off) return fail(c, DAGRT_EINVAL, "range out of bounds");
  if (bytes && !dst) return fail(c, DAGRT_EINVAL, "null dst");
  // a read that needs a copy orders the copy after its producers on the D2H
  // stream (one host round trip); otherwise the host waits on the events
  const bool copy = bytes && (!a->host || a->coh == COH_DEVICE) && c->be->real() && !a->managed;
  if (c->cfg.policy != DAGRT_SERIAL_SYNC)
    if (dagrt_status s = host_sync_parents(c, a, false, copy ? c->d2h_stream : nullptr)) return s;
  if (!a->host) return d2h(c, a, off, bytes, dst);
  if (a->managed) a->host_touched = true;
  if (a->coh == COH_DEVICE) {
    if (dagrt_status s = d2h(c, a, off, bytes, a->host + off)) return s;
    if (off == 0 && bytes == a->bytes) a->coh = COH_BOTH;
  }
  if (bytes && dst != a->host + off) memcpy(dst, a->host + off, bytes);
  return DAGRT_OK;
}

static dagrt_status host_write_prepare(dagrt_ctx c, ArrayRec* a, bool whole) {
  if (c->cfg.policy != DAGRT_SERIAL_SYNC) {
    if (dagrt_status s = host_sync_parents(c, a, true)) return s;
  }
  if (a->managed) a->host_touched = true;
  if (a->h2d_pending) {  // the copy engine may still read the mirror
    CK(c->be->event_sync(a->h2d_ev), "cudaEventSynchronize copy");
    a->h2d_pending = false;
  }
  if (a->host && a->coh == COH_DEVICE && !whole)
    if (dagrt_status s = d2h(c, a, 0, a->bytes, a->host)) return s;
  return DAGRT_OK;
}

dagrt_status dagrt_host_write(dagrt_ctx c, dagrt_array h, size_t off, size_t bytes,
                              const void* src) {
  NvtxRange nvtx_("dagrt_host_write");
  GUARD(c);
  ArrayRec* a = get_array(c, h);
  if (!a) return fail(c, DAGRT_ENOTFOUND, "array handle");
  if (off > a->bytes || bytes > a->bytes - off) return fail(c, DAGRT_EINVAL, "range out of bounds");
  if (bytes && !src) return fail(c, DAGRT_EINVAL, "null src");
  bool whole = off == 0 && bytes == a->bytes;
  if (dagrt_status s = host_write_prepare(c, a, whole)) return s;
  a->last_writer = -1;
  a->readers.clear();
  if (!a->host) {
    if (!bytes) return DAGRT_OK;
    trace_op(c, DAGRT_OP_H2D, -1, array_index(c, a), (int64_t)off, bytes);
    c->st.h2d_bytes += bytes;
    c->st.h2d_copies++;
    if (c->be->real()) {
      CK(c->be->copy_async(a->dev + off, src, bytes, cudaMemcpyHostToDevice, c->copy_stream),
         "cudaMemcpyAsync H2D");
      CK(c->be->stream_sync(c->copy_stream), "cudaStreamSynchronize");
      c->st.host_syncs++;
    }
    return DAGRT_OK;
  }
  if (bytes && src != a->host + off) memcpy(a->host + off, src, bytes);
  a->coh = COH_HOST;
  return DAGRT_OK;
}

dagrt_status dagrt_host_map(dagrt_ctx c, dagrt_array h, int32_t access, void** host_ptr) {
  NvtxRange nvtx_("dagrt_host_map");
  GUARD(c);
  ArrayRec* a = get_array(c, h);
  if (!a) return fail(c, DAGRT_ENOTFOUND, "array handle");
  if (!host_ptr || access < DAGRT_R || access > DAGRT_RW) return fail(c, DAGRT_EINVAL, "bad access/ptr");
  if (!a->host) return fail(c, DAGRT_ESTATE, "array has no host mirror");
  if (access & DAGRT_W) {
    // a W map is a host write of the whole array; RW keeps the current data
    if (dagrt_status s = host_write_prepare(c, a, !(access & DAGRT_R))) return s;
    if ((access & DAGRT_R) && a->coh == COH_DEVICE) {
      if (dagrt_status s = d2h(c, a, 0, a->bytes, a->host)) return s;
    }
    a->last_writer = -1;
    a->readers.clear();
    a->coh = COH_HOST;
  } else {
    const bool copy = a->bytes && a->coh == COH_DEVICE && c->be->real() && !a->managed;
    if (c->cfg.policy != DAGRT_SERIAL_SYNC)
      if (dagrt_status s = host_sync_parents(c, a, false, copy ? c->d2h_stream : nullptr)) return s;
    if (a->coh == COH_DEVICE) {
      if (dagrt_status s = d2h(c, a, 0, a->bytes, a->host)) return s;
      a->coh = COH_BOTH;
    }
  }
  a->mapped = true;
  if (a->managed) a->host_touched = true;
  *host_ptr = a->host;
  return DAGRT_OK;
}

dagrt_status dagrt_host_unmap(dagrt_ctx c, dagrt_array h) {
  GUARD(c);
  ArrayRec* a = get_array(c, h);
  if (!a) return fail(c, DAGRT_ENOTFOUND, "array handle");
  if (!a->mapped) return fail(c, DAGRT_ESTATE, "array not mapped");
  a->mapped = false;
  return DAGRT_OK;
}

dagrt_status dagrt_sync(dagrt_ctx c) {
  NvtxRange nvtx_("dagrt_sync");
  GUARD(c);
  for (size_t s = 0; s < c->streams.size(); ++s) {
    trace_op(c, DAGRT_OP_STREAM_SYNC, (int32_t)s, 0, 0, 0);
    CK(c->be->stream_sync(c->streams[s].s), "cudaStreamSynchronize");
  }
  for (void* s : {c->copy_stream, c->d2h_stream, c->graph_stream, c->serial_stream})
    CK(c->be->stream_sync(s), "cudaStreamSynchronize");
  c->st.host_syncs++;
  retire_all(c);
  recycle(c);
  tune_collect(c);
  for (size_t i = 1; i < c->arrays.size(); ++i) c->arrays[i].h2d_pending = false;
  return DAGRT_OK;
}

dagrt_status dagrt_dag_export(dagrt_ctx c, dagrt_vertex_info* v, uint32_t* nv, dagrt_edge_info* e,
                              uint32_t* ne) {
  GUARD(c);
  if (!nv || !ne) return fail(c, DAGRT_EINVAL, "null counts");
  uint32_t cv = *nv, ce = *ne;
  *nv = (uint32_t)c->rec_v.size();
  *ne = (uint32_t)c->rec_e.size();
  if (!v && !e) return DAGRT_OK;
  if (cv < *nv || ce < *ne) return fail(c, DAGRT_EINVAL, "capacity");
  if (v) std::copy(c->rec_v.begin(), c->rec_v.end(), v);
  if (e) std::copy(c->rec_e.begin(), c->rec_e.end(), e);
  return DAGRT_OK;
}

dagrt_status dagrt_dag_clear(dagrt_ctx c) {
  GUARD(c);
  c->rec_v.clear();
  c->rec_e.clear();
  c->trace.clear();
  return DAGRT_OK;
}

dagrt_status dagrt_trace_export(dagrt_ctx c, dagrt_trace_op* ops, uint32_t* n) {
  GUARD(c);
  if (!n) return fail(c, DAGRT_EINVAL, "null n");
  uint32_t cap = *n;
  *n = (uint32_t)c->trace.size();
  if (!ops) return DAGRT_OK;
  if (cap < *n) return fail(c, DAGRT_EINVAL, "capacity");
  std::copy(c->trace.begin(), c->trace.end(), ops);
  return DAGRT_OK;
}

dagrt_status dagrt_stats(dagrt_ctx c, void* out, size_t size) {
  if (!c || !out) return DAGRT_EINVAL;
  c->st.graph_replays = c->be->replays;
  c->st.graph_captures = c->be->captures;
  c->st.eager_batches = c->be->eager;
  c->st.table_vertices = c->vertices.size();
  c->st.epoch_base = (uint64_t)c->vid_base;
  c->st.max_readers = 0;
  for (size_t i = 1; i < c->arrays.size(); ++i)
    if (c->arrays[i].live) c->st.max_readers = std::max<uint64_t>(c->st.max_readers, c->arrays[i].readers.size());
  memcpy(out, &c->st, std::min(size, sizeof(dagrt_stats_t)));
  return DAGRT_OK;
}

dagrt_status dagrt_stats_reset(dagrt_ctx c) {
  if (!c) return DAGRT_EINVAL;
  c->st = dagrt_stats_t{};
  c->be->replays = c->be->captures = c->be->eager = 0;
  c->st.streams = c->streams.size();
  return DAGRT_OK;
}

dagrt_status dagrt_stream_count(dagrt_ctx c, int32_t* n) {
  if (!c || !n) return DAGRT_EINVAL;
  *n = (int32_t)c->streams.size();
  return DAGRT_OK;
}

dagrt_status dagrt_stream_handle(dagrt_ctx c, int32_t i, void** s) {
  if (!c || !s) return DAGRT_EINVAL;
  if (i == -2) { *s = c->copy_stream; return DAGRT_OK; }
  if (i == -3) { *s = c->serial_stream; return DAGRT_OK; }
  if (i == -4) { *s = c->graph_stream; return DAGRT_OK; }
  if (i < 0 || (size_t)i >= c->streams.size()) return DAGRT_EINVAL;
  *s = c->streams[i].s;
  return DAGRT_OK;
}

dagrt_status dagrt_profile_enable(dagrt_ctx c, dagrt_kernel kh, int32_t on) {
  GUARD(c);
  KernelRec* k;
  if (dagrt_status s = lookup_kernel(c, kh, &k)) return s;
  k->prof = on != 0;
  // per-launch timing events are not replayable: no deferral while profiling
  bool any = false;
  for (const KernelRec& kr : c->kernels) any = any || kr.prof;
  if (cudaError_t e = c->be->flush()) return cuda_fail(c, e, "flush");
  c->be->enabled = c->cfg.graph_cache && c->cfg.policy != DAGRT_SERIAL_SYNC && c->be->real() &&
                   !any && !c->timeline;
  return DAGRT_OK;
}

dagrt_status dagrt_profile_collect(dagrt_ctx c, dagrt_kernel kh, int32_t* count, double* sum_ms,
                                   double* busy_ms) {
  GUARD(c);
  if (!count || !sum_ms || !busy_ms) return fail(c, DAGRT_EINVAL, "null out");
  *count = 0;
  *sum_ms = 0.0;
  *busy_ms = 0.0;
  std::vector<std::pair<double, double>> iv;
  void* ref = nullptr;
  std::vector<ProfRec> keep;
  for (const ProfRec& p : c->prof) {
    if (p.kernel != kh) { keep.push_back(p); continue; }
    CK(c->be->event_sync(p.ev1), "cudaEventSynchronize profile");
    if (!ref) ref = p.ev0;
    float a = 0.f, b = 0.f, d = 0.f;
    CK(c->be->elapsed(&a, ref, p.ev0), "cudaEventElapsedTime");
    CK(c->be->elapsed(&b, ref, p.ev1), "cudaEventElapsedTime");
    CK(c->be->elapsed(&d, p.ev0, p.ev1), "cudaEventElapsedTime");
    iv.push_back({a, b});
    *sum_ms += d;
    (*count)++;
    c->tev_pool.push_back(p.ev0);
    c->tev_pool.push_back(p.ev1);
  }
  c->prof.swap(keep);
  std::sort(iv.begin(), iv.end());
  double cs = 0, ce = -1e300;
  for (auto& x : iv) {
    if (x.first > ce) {
      if (ce > -1e300) *busy_ms += ce - cs;
      cs = x.first;
      ce = x.second;
    } else if (x.second > ce) {
      ce = x.second;
    }
  }
  if (ce > -1e300) *busy_ms += ce - cs;
  return DAGRT_OK;
}

dagrt_status dagrt_timeline_enable(dagrt_ctx c, int32_t on) {
  GUARD(c);
  c->timeline = on != 0;
  if (cudaError_t e = c->be->flush()) return cuda_fail(c, e, "flush");
  bool any = false;
  for (const KernelRec& kr : c->kernels) any = any || kr.prof;
  c->be->enabled = c->cfg.graph_cache && c->cfg.policy != DAGRT_SERIAL_SYNC && c->be->real() &&
                   !any && !c->timeline;
  return DAGRT_OK;
}

dagrt_status dagrt_timeline_export(dagrt_ctx c, dagrt_timeline_rec* recs, uint32_t* n) {
  GUARD(c);
  if (!n) return fail(c, DAGRT_EINVAL, "null n");
  uint32_t cap = *n;
  *n = (uint32_t)c->tl.size();
  if (!recs) return DAGRT_OK;
  if (cap < *n) return fail(c, DAGRT_EINVAL, "capacity");
  void* ref = c->tl.empty() ? nullptr : c->tl[0].ev0;
  for (size_t i = 0; i < c->tl.size(); ++i) {
    TimeRec& r = c->tl[i];
    CK(c->be->event_sync(r.ev1), "cudaEventSynchronize timeline");
    float a = 0.f, b = 0.f;
    CK(c->be->elapsed(&a, ref, r.ev0), "cudaEventElapsedTime");
    CK(c->be->elapsed(&b, ref, r.ev1), "cudaEventElapsedTime");
    recs[i] = dagrt_timeline_rec{r.kind, r.stream, r.vertex, r.id, r.bytes, a, b};
  }
  for (TimeRec& r : c->tl) {
    c->tev_pool.push_back(r.ev0);
    c->tev_pool.push_back(r.ev1);
  }
  c->tl.clear();
  return DAGRT_OK;
}

dagrt_status dagrt_launch_raw(dagrt_ctx c, dagrt_kernel kh, dagrt_dim3 grid, dagrt_dim3 block,
                              uint32_t smem, const dagrt_arg* args, int32_t nargs, void* stream) {
  GUARD(c);
  KernelRec* k;
  if (dagrt_status s = lookup_kernel(c, kh, &k)) return s;
  uint64_t vals[kMaxArgs + 1];
  void* argv[kMaxArgs + 1];
  ArrayRec* arrs[kMaxArgs];
  if (dagrt_status s = marshal(c, *k, args, nargs, vals, argv, arrs, dim3(grid.x, grid.y, grid.z),
                               dim3(block.x, block.y, block.z), smem))
    return s;
  CK(c->be->launch_now(k->fn, dim3(grid.x, grid.y, grid.z), dim3(block.x, block.y, block.z), argv, smem,
                   stream, k->coop),
     "cudaLaunchKernel raw");
  return DAGRT_OK;
}

// ------------------------------------------------------------ manual CUDA graphs
dagrt_status dagrt_graph_create(dagrt_ctx c, dagrt_graph* g) {
  GUARD(c);
  if (!g) return fail(c, DAGRT_EINVAL, "null graph out");
  if (!c->be->real()) return fail(c, DAGRT_ESTATE, "graphs need the CUDA backend");
  auto* gr = new (std::nothrow) dagrt_graph_s();
  if (!gr) return DAGRT_ENOMEM;
  CK(cudaGraphCreate(&gr->r.g, 0), "cudaGraphCreate");
  c->graphs.push_back(gr);
  *g = gr;
  return DAGRT_OK;
}

static dagrt_status graph_deps(dagrt_ctx c, dagrt_graph g, const uint32_t* deps, int32_t ndeps,
                               std::vector<cudaGraphNode_t>* out) {
  for (int i = 0; i < ndeps; ++i) {
    if (deps[i] >= g->r.nodes.size()) return fail(c, DAGRT_EINVAL, "bad dependency node %u", deps[i]);
    out->push_back(g->r.nodes[deps[i]]);
  }
  return DAGRT_OK;
}

dagrt_status dagrt_graph_add_kernel(dagrt_ctx c, dagrt_graph g, dagrt_kernel kh, dagrt_dim3 grid,
                                    dagrt_dim3 block, uint32_t smem, const dagrt_arg* args,
                                    int32_t nargs, const uint32_t* deps, int32_t ndeps,
                                    uint32_t* node) {
  GUARD(c);
  if (!g || !node) return fail(c, DAGRT_EINVAL, "null graph/node");
  KernelRec* k;
  if (dagrt_status s = lookup_kernel(c, kh, &k)) return s;
  if (builtin_resolver(k->fn))
    return fail(c, DAGRT_EINVAL, "experimental built-ins (libdagrt_exp.so) are not graph nodes");
  uint64_t vals[kMaxArgs + 1];
  void* argv[kMaxArgs + 1];
  ArrayRec* arrs[kMaxArgs];
  if (dagrt_status s = marshal(c, *k, args, nargs, vals, argv, arrs, dim3(grid.x, grid.y, grid.z),
                               dim3(block.x, block.y, block.z), smem))
    return s;
  std::vector<cudaGraphNode_t> d;
  if (dagrt_status s = graph_deps(c, g, deps, ndeps, &d)) return s;
  cudaKernelNodeParams p{};
  p.func = const_cast<void*>(k->fn);
  p.gridDim = dim3(grid.x, grid.y, grid.z);
  p.blockDim = dim3(block.x, block.y, block.z);
  p.sharedMemBytes = smem;
  p.kernelParams = argv;
  cudaGraphNode_t n;
  CK(cudaGraphAddKernelNode(&n, g->r.g, d.data(), d.size(), &p), "cudaGraphAddKernelNode");
  if (k->coop) {  // co-residency guaranteed in the graph too (grid barrier kernels)
    cudaLaunchAttributeValue v{};
    v.cooperative = 1;
    CK(cudaGraphKernelNodeSetAttribute(n, cudaLaunchAttributeCooperative, &v),
       "cudaGraphKernelNodeSetAttribute cooperative");
  }
  g->r.nodes.push_back(n);
  *node = (uint32_t)g->r.nodes.size() - 1;
  return DAGRT_OK;
}

dagrt_status dagrt_graph_add_copy(dagrt_ctx c, dagrt_graph g, dagrt_array h, int32_t dir, size_t off,
                                  size_t bytes, const uint32_t* deps, int32_t ndeps, uint32_t* node) {
  GUARD(c);
  if (!g || !node) return fail(c, DAGRT_EINVAL, "null graph/node");
  ArrayRec* a = get_array(c, h);
  if (!a) return fail(c, DAGRT_ENOTFOUND, "array handle");
  if (!a->host) return fail(c, DAGRT_ESTATE, "array has no host mirror");
  if (off > a->bytes || bytes > a->bytes - off) return fail(c, DAGRT_EINVAL, "range");
  std::vector<cudaGraphNode_t> d;
  if (dagrt_status s = graph_deps(c, g, deps, ndeps, &d)) return s;
  cudaGraphNode_t n;
  if (dir == 0)
    CK(cudaGraphAddMemcpyNode1D(&n, g->r.g, d.data(), d.size(), a->dev + off, a->host + off, bytes,
                                cudaMemcpyHostToDevice), "cudaGraphAddMemcpyNode1D");
  else
    CK(cudaGraphAddMemcpyNode1D(&n, g->r.g, d.data(), d.size(), a->host + off, a->dev + off, bytes,
                                cudaMemcpyDeviceToHost), "cudaGraphAddMemcpyNode1D");
  g->r.nodes.push_back(n);
  *node = (uint32_t)g->r.nodes.size() - 1;
  return DAGRT_OK;
}

dagrt_status dagrt_graph_add_read(dagrt_ctx c, dagrt_graph g, dagrt_array h, size_t off, size_t bytes,
                                  void* dst, const uint32_t* deps, int32_t ndeps, uint32_t* node) {
  GUARD(c);
  if (!g || !node || !dst) return fail(c, DAGRT_EINVAL, "null graph/node/dst");
  ArrayRec* a = get_array(c, h);
  if (!a) return fail(c, DAGRT_ENOTFOUND, "array handle");
  if (off > a->bytes || bytes > a->bytes - off) return fail(c, DAGRT_EINVAL, "range");
  std::vector<cudaGraphNode_t> d;
  if (dagrt_status s = graph_deps(c, g, deps, ndeps, &d)) return s;
  cudaGraphNode_t n;
  CK(cudaGraphAddMemcpyNode1D(&n, g->r.g, d.data(), d.size(), dst, a->dev + off, bytes,
                              cudaMemcpyDeviceToHost), "cudaGraphAddMemcpyNode1D");
  g->r.nodes.push_back(n);
  *node = (uint32_t)g->r.nodes.size() - 1;
  return DAGRT_OK;
}

dagrt_status dagrt_graph_instantiate(dagrt_ctx c, dagrt_graph g) {
  GUARD(c);
  if (!g) return fail(c, DAGRT_EINVAL, "null graph");
  if (g->r.exec) { cudaGraphExecDestroy(g->r.exec); g->r.exec = nullptr; }
  CK(cudaGraphInstantiate(&g->r.exec, g->r.g, 0), "cudaGraphInstantiate");
  CK(cudaGraphUpload(g->r.exec, (cudaStream_t)c->graph_stream), "cudaGraphUpload");
  return DAGRT_OK;
}

dagrt_status dagrt_graph_run(dagrt_ctx c, dagrt_graph g, int32_t wait) {
  NvtxRange nvtx_("dagrt_graph_run");
  GUARD(c);
  if (!g || !g->r.exec) return fail(c, DAGRT_ESTATE, "graph not instantiated");
  CK(cudaGraphLaunch(g->r.exec, (cudaStream_t)c->graph_stream), "cudaGraphLaunch");
  if (wait) CK(cudaStreamSynchronize((cudaStream_t)c->graph_stream), "cudaStreamSynchronize graph");
  return DAGRT_OK;
}

dagrt_status dagrt_graph_destroy(dagrt_ctx c, dagrt_graph g) {
  if (!c || !g) return DAGRT_EINVAL;
  auto it = std::find(c->graphs.begin(), c->graphs.end(), g);
  if (it == c->graphs.end()) return DAGRT_ENOTFOUND;
  if (g->r.exec) cudaGraphExecDestroy(g->r.exec);
  if (g->r.g) cudaGraphDestroy(g->r.g);
  delete g;
  c->graphs.erase(it);
  return DAGRT_OK;
}

}  // extern "C"
