// Multi-GPU DAG placement (§VII, the
// paper's future work: "compute data location and migration costs at run
// time" to schedule one application over several GPUs).
//
// A layer over per-slot scheduler contexts (runtime.cpp), written against the
// public C ABI only (include/dagrt.h "multi-GPU placement"): every launch is
// placed on one slot and becomes a vertex of that slot's DAG, where the
// single-GPU scheduler infers its dependencies, stream and event waits.
// Cross-slot edges are data migrations expressed as library-call vertices
// (dagrt_launch_library), so the per-slot schedulers order them against
// their own readers and writers:
//
//   slot d  "migrate_pre"  (replica on d, W)  records ev_pre[d] after d's users
//   slot s  "migrate_out"  (replica on s, R)  waits ev_pre[d], peer copy s -> d,
//                                             records ev_done[s]
//   slot d  "migrate_in"   (replica on d, W)  waits ev_done[s]
//
// One event per slot and role suffices: cudaStreamWaitEvent binds to the
// record current when it is called, and the three vertices are enqueued in
// host order before the event is recorded again.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/dagrt.h"

namespace {

constexpr int kMaxSlots = 16;
constexpr int kMaxArgs = 16;
constexpr uint64_t kHostBit = 1ull << 63;
// bandwidth model of the placement estimate (GB/s = 1e3 bytes/us): B200 HBM3e,
// NVLink 5 per direction, a copy within one device, PCIe Gen5 host link
constexpr double kHbmGBs = 6500.0, kPeerGBs = 700.0, kSameDevGBs = 3000.0, kHostGBs = 50.0;

struct Replica {
  void* dev = nullptr;
  dagrt_array h = 0;
  bool owned = false;
  void* up_ev = nullptr;  // last upload from the host mirror into this replica
};

struct MArray {
  size_t bytes = 0;
  char* host = nullptr;
  int home = 0;
  uint64_t valid = 0;       // bit s: slot s's replica is current; kHostBit: the mirror is
  uint64_t uploading = 0;   // slots with an upload from the mirror possibly in flight
  uint32_t gen = 0;
  bool live = false;
  std::vector<Replica> rep;
};

struct Slot {
  int dev = 0;
  dagrt_ctx ctx = nullptr;
  double busy_us = 0.0;  // estimated completion of the work placed here since the last sync
  void* ev_pre = nullptr;
  void* ev_done = nullptr;
};

struct KernelEntry {
  std::string name;
  std::vector<dagrt_kernel> h;  // per slot
  std::vector<int32_t> kinds;
};

// ---- library-call bodies (run on the stream the slot's scheduler picked)
struct RecordJob {
  void* ev;
};
int32_t cb_record(void* s, void* u) {
  return cudaEventRecord((cudaEvent_t)static_cast<RecordJob*>(u)->ev, (cudaStream_t)s) == cudaSuccess ? 0 : 1;
}
struct WaitJob {
  void* ev;
};
int32_t cb_wait(void* s, void* u) {
  return cudaStreamWaitEvent((cudaStream_t)s, (cudaEvent_t)static_cast<WaitJob*>(u)->ev, 0) == cudaSuccess ? 0 : 1;
}
struct CopyJob {
  void* wait_ev;
  void* done_ev;
  void* dst;
  int ddev;
  const void* src;
  int sdev;
  size_t bytes;
  bool from_host;
};
int32_t cb_copy(void* s, void* u) {
  const CopyJob* j = static_cast<CopyJob*>(u);
  cudaStream_t st = (cudaStream_t)s;
  if (j->wait_ev && cudaStreamWaitEvent(st, (cudaEvent_t)j->wait_ev, 0) != cudaSuccess) return 1;
  if (j->bytes) {
    cudaError_t e;
    if (j->from_host) e = cudaMemcpyAsync(j->dst, j->src, j->bytes, cudaMemcpyHostToDevice, st);
    else if (j->ddev == j->sdev) e = cudaMemcpyAsync(j->dst, j->src, j->bytes, cudaMemcpyDeviceToDevice, st);
    else e = cudaMemcpyPeerAsync(j->dst, j->ddev, j->src, j->sdev, j->bytes, st);
    if (e != cudaSuccess) return 2;
  }
  if (j->done_ev && cudaEventRecord((cudaEvent_t)j->done_ev, st) != cudaSuccess) return 3;
  return 0;
}

}  // namespace

struct dagrt_multi_s {
  std::vector<Slot> slots;
  std::vector<MArray> arrays;  // index 0 unused
  std::vector<KernelEntry> kernels;
  int placement = DAGRT_PLACE_DATA;
  bool real = true;
  std::string err;
  uint64_t rr = 0;
  uint64_t fake_next = 1ull << 44;  // RECORD backend: distinct fake replica addresses
  dagrt_multi_stats_t st{};
};

namespace {

dagrt_status mfail(dagrt_multi m, dagrt_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  m->err = buf;
  return s;
}

// forward a slot context's failure with its message
dagrt_status slot_fail(dagrt_multi m, int s, dagrt_status st, const char* what) {
  const char* e = dagrt_last_error(m->slots[s].ctx);
  return mfail(m, st, "slot %d %s: %s", s, what, e ? e : "");
}

dagrt_status set_dev(dagrt_multi m, int s) {
  if (!m->real) return DAGRT_OK;
  cudaError_t e = cudaSetDevice(m->slots[s].dev);
  if (e != cudaSuccess) return mfail(m, DAGRT_ECUDA, "cudaSetDevice(%d): %s", m->slots[s].dev, cudaGetErrorName(e));
  return DAGRT_OK;
}

dagrt_status new_event(dagrt_multi m, int s, void** ev) {
  *ev = nullptr;
  if (!m->real) return DAGRT_OK;
  if (dagrt_status r = set_dev(m, s)) return r;
  cudaEvent_t e;
  cudaError_t c = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (c != cudaSuccess) return mfail(m, DAGRT_ECUDA, "cudaEventCreate: %s", cudaGetErrorName(c));
  *ev = (void*)e;
  return DAGRT_OK;
}

MArray* get(dagrt_multi m, dagrt_marray h) {
  const uint32_t idx = (uint32_t)(h & 0xffffffffu), gen = (uint32_t)(h >> 32);
  if (idx == 0 || idx >= m->arrays.size()) return nullptr;
  MArray* a = &m->arrays[idx];
  return a->live && a->gen == gen ? a : nullptr;
}

inline uint64_t bit(int s) { return 1ull << s; }

// The replica of a on slot s, allocated and registered on first use.
dagrt_status ensure_replica(dagrt_multi m, MArray* a, int s) {
  Replica& r = a->rep[s];
  if (r.h) return DAGRT_OK;
  if (dagrt_status e = set_dev(m, s)) return e;
  const size_t alloc = a->bytes ? a->bytes : 16;
  if (m->real) {
    cudaError_t e = cudaMalloc(&r.dev, alloc);
    if (e != cudaSuccess) return mfail(m, DAGRT_ECUDA, "replica of %zu bytes on slot %d: %s", a->bytes, s, cudaGetErrorName(e));
  } else {
    r.dev = (void*)(uintptr_t)m->fake_next;
    m->fake_next += (alloc + 4095) & ~(size_t)4095;
  }
  r.owned = true;
  if (dagrt_status e = dagrt_array_register(m->slots[s].ctx, r.dev, nullptr, a->bytes, &r.h)) {
    if (m->real) cudaFree(r.dev);
    r.dev = nullptr;
    return slot_fail(m, s, e, "replica register");
  }
  m->st.replicas++;
  m->st.bytes_replicas += a->bytes;
  return DAGRT_OK;
}

// Link bandwidth (GB/s) of a copy of a current copy of `a` to slot d, and the
// source slot (-1: the host mirror, -2: no current copy anywhere).
double source_of(dagrt_multi m, const MArray* a, int d, int* src) {
  const int n = (int)m->slots.size();
  int best = -2;
  double bw = 0.0;
  for (int s = 0; s < n; ++s) {
    if (!(a->valid & bit(s))) continue;
    const double b = m->slots[s].dev == m->slots[d].dev ? kSameDevGBs : kPeerGBs;
    if (b > bw || (b == bw && s == a->home)) {
      bw = b;
      best = s;
    }
  }
  if (best < 0 && (a->valid & kHostBit) && a->host) {
    best = -1;
    bw = kHostGBs;
  }
  *src = best;
  return bw;
}

// Make a's copy on slot d current (the three migration vertices, or an upload).
dagrt_status migrate(dagrt_multi m, MArray* a, int d) {
  if (a->valid & bit(d)) return DAGRT_OK;
  if (dagrt_status e = ensure_replica(m, a, d)) return e;
  int s;
  source_of(m, a, d, &s);
  Slot& D = m->slots[d];
  Replica& rd = a->rep[d];
  if (s >= 0) {
    Slot& S = m->slots[s];
    Replica& rs = a->rep[s];
    RecordJob pre{D.ev_pre};
    int32_t w = DAGRT_W, r = DAGRT_R;
    if (dagrt_status e = set_dev(m, d)) return e;
    if (dagrt_status e = dagrt_launch_library(D.ctx, cb_record, &pre, "migrate_pre", &rd.h, &w, 1))
      return slot_fail(m, d, e, "migrate_pre");
    CopyJob cj{D.ev_pre, S.ev_done, rd.dev, D.dev, rs.dev, S.dev, a->bytes, false};
    if (dagrt_status e = set_dev(m, s)) return e;
    if (dagrt_status e = dagrt_launch_library(S.ctx, cb_copy, &cj, "migrate_out", &rs.h, &r, 1))
      return slot_fail(m, s, e, "migrate_out");
    WaitJob wj{S.ev_done};
    if (dagrt_status e = set_dev(m, d)) return e;
    if (dagrt_status e = dagrt_launch_library(D.ctx, cb_wait, &wj, "migrate_in", &rd.h, &w, 1))
      return slot_fail(m, d, e, "migrate_in");
    m->st.migrations_peer++;
    m->st.bytes_peer += a->bytes;
  } else if (s == -1) {
    if (!rd.up_ev)
      if (dagrt_status e = new_event(m, d, &rd.up_ev)) return e;
    CopyJob cj{nullptr, rd.up_ev, rd.dev, D.dev, a->host, -1, a->bytes, true};
    int32_t w = DAGRT_W;
    if (dagrt_status e = set_dev(m, d)) return e;
    if (dagrt_status e = dagrt_launch_library(D.ctx, cb_copy, &cj, "upload", &rd.h, &w, 1))
      return slot_fail(m, d, e, "upload");
    a->uploading |= bit(d);
    m->st.migrations_host++;
    m->st.bytes_host += a->bytes;
  }  // s == -2: nothing current anywhere (never written): the replica is as good as any
  a->valid |= bit(d);
  return DAGRT_OK;
}

KernelEntry* kernel_of(dagrt_multi m, const char* name) {
  for (KernelEntry& k : m->kernels)
    if (k.name == name) return &k;
  KernelEntry k;
  k.name = name;
  for (size_t s = 0; s < m->slots.size(); ++s) {
    dagrt_kernel h;
    if (dagrt_kernel_lookup(m->slots[s].ctx, name, &h) != DAGRT_OK) {
      mfail(m, DAGRT_ENOTFOUND, "no kernel named '%s'", name);
      return nullptr;
    }
    k.h.push_back(h);
  }
  int32_t kinds[kMaxArgs], n = kMaxArgs;
  if (dagrt_kernel_signature(m->slots[0].ctx, k.h[0], kinds, &n) != DAGRT_OK) {
    mfail(m, DAGRT_ESIG, "signature of '%s'", name);
    return nullptr;
  }
  k.kinds.assign(kinds, kinds + n);
  m->kernels.push_back(k);
  return &m->kernels.back();
}

inline bool is_ptr(int32_t k) { return k == 2 || k == 3 || k == 4; }
inline bool reads(int32_t k) { return k == 2 || k == 3; }
inline bool writes(int32_t k) { return k == 3 || k == 4; }

}  // namespace

extern "C" {

dagrt_status dagrt_multi_create(const int32_t* devices, int32_t n, const dagrt_config* cfg, int32_t placement,
                                dagrt_multi* out) {
  if (!devices || !out || n < 1 || n > kMaxSlots) return DAGRT_EINVAL;
  if (placement != DAGRT_PLACE_DATA && placement != DAGRT_PLACE_ROUND_ROBIN) return DAGRT_EINVAL;
  dagrt_multi m = new (std::nothrow) dagrt_multi_s();
  if (!m) return DAGRT_ENOMEM;
  m->placement = placement;
  m->real = !cfg || cfg->backend == DAGRT_BACKEND_CUDA;
  m->arrays.resize(1);
  m->slots.resize(n);
  for (int s = 0; s < n; ++s) {
    m->slots[s].dev = devices[s];
    if (dagrt_status e = dagrt_create(devices[s], cfg, &m->slots[s].ctx)) {
      dagrt_multi_destroy(m);
      return e;
    }
    if (new_event(m, s, &m->slots[s].ev_pre) || new_event(m, s, &m->slots[s].ev_done)) {
      dagrt_multi_destroy(m);
      return DAGRT_ECUDA;
    }
  }
  if (m->real)  // NVLink peer access between distinct devices (copies work without it, staged)
    for (int s = 0; s < n; ++s)
      for (int t = 0; t < n; ++t) {
        if (m->slots[s].dev == m->slots[t].dev) continue;
        int ok = 0;
        if (cudaDeviceCanAccessPeer(&ok, m->slots[s].dev, m->slots[t].dev) == cudaSuccess && ok) {
          cudaSetDevice(m->slots[s].dev);
          cudaDeviceEnablePeerAccess(m->slots[t].dev, 0);  // already enabled: harmless error
        }
        cudaGetLastError();
      }
  *out = m;
  return DAGRT_OK;
}

dagrt_status dagrt_multi_destroy(dagrt_multi m) {
  if (!m) return DAGRT_EINVAL;
  for (size_t s = 0; s < m->slots.size(); ++s)
    if (m->slots[s].ctx) {
      set_dev(m, (int)s);
      dagrt_sync(m->slots[s].ctx);
    }
  for (size_t s = 0; s < m->slots.size(); ++s)
    if (m->slots[s].ctx) {
      set_dev(m, (int)s);
      dagrt_destroy(m->slots[s].ctx);
    }
  for (MArray& a : m->arrays)
    for (size_t s = 0; s < a.rep.size(); ++s) {
      set_dev(m, (int)s);
      if (m->real && a.rep[s].owned && a.rep[s].dev) cudaFree(a.rep[s].dev);
      if (a.rep[s].up_ev) cudaEventDestroy((cudaEvent_t)a.rep[s].up_ev);
    }
  for (size_t s = 0; s < m->slots.size(); ++s) {
    set_dev(m, (int)s);
    if (m->slots[s].ev_pre) cudaEventDestroy((cudaEvent_t)m->slots[s].ev_pre);
    if (m->slots[s].ev_done) cudaEventDestroy((cudaEvent_t)m->slots[s].ev_done);
  }
  delete m;
  return DAGRT_OK;
}

const char* dagrt_multi_last_error(dagrt_multi m) { return m ? m->err.c_str() : "null multi-context"; }

dagrt_status dagrt_multi_slot_ctx(dagrt_multi m, int32_t slot, dagrt_ctx* out) {
  if (!m || !out) return DAGRT_EINVAL;
  if (slot < 0 || slot >= (int32_t)m->slots.size()) return mfail(m, DAGRT_EINVAL, "slot %d out of range", slot);
  *out = m->slots[slot].ctx;
  return DAGRT_OK;
}

dagrt_status dagrt_multi_array_register(dagrt_multi m, int32_t home, void* dev, void* host_pinned, size_t bytes,
                                        dagrt_marray* out) {
  if (!m || !out) return DAGRT_EINVAL;
  if (home < 0 || home >= (int32_t)m->slots.size()) return mfail(m, DAGRT_EINVAL, "home slot %d out of range", home);
  MArray a;
  a.bytes = bytes;
  a.host = static_cast<char*>(host_pinned);
  a.home = home;
  a.rep.resize(m->slots.size());
  a.live = true;
  size_t idx = 1;
  while (idx < m->arrays.size() && m->arrays[idx].live) ++idx;
  a.gen = idx < m->arrays.size() ? m->arrays[idx].gen + 1 : 1;
  if (dev) {
    if (dagrt_status e = set_dev(m, home)) return e;
    if (dagrt_status e = dagrt_array_register(m->slots[home].ctx, dev, nullptr, bytes, &a.rep[home].h))
      return slot_fail(m, home, e, "array register");
    a.rep[home].dev = dev;
    a.valid = bit(home);
  } else if (host_pinned) {
    a.valid = kHostBit;
  }
  if (idx < m->arrays.size()) m->arrays[idx] = a;
  else m->arrays.push_back(a);
  *out = ((uint64_t)a.gen << 32) | idx;
  return DAGRT_OK;
}

dagrt_status dagrt_multi_array_ptr(dagrt_multi m, dagrt_marray h, int32_t slot, void** dev) {
  if (!m || !dev) return DAGRT_EINVAL;
  MArray* a = get(m, h);
  if (!a) return mfail(m, DAGRT_ENOTFOUND, "stale multi-array handle");
  if (slot < 0 || slot >= (int32_t)m->slots.size()) return mfail(m, DAGRT_EINVAL, "slot %d out of range", slot);
  *dev = a->rep[slot].dev;
  return DAGRT_OK;
}

dagrt_status dagrt_multi_launch(dagrt_multi m, const char* name, dagrt_dim3 grid, dagrt_dim3 block, uint32_t smem,
                                const dagrt_arg* args, int32_t nargs, int32_t slot, int32_t* placed) {
  if (!m || !name || (nargs > 0 && !args)) return DAGRT_EINVAL;
  const int n = (int)m->slots.size();
  if (slot >= n) return mfail(m, DAGRT_EINVAL, "slot %d out of range", slot);
  KernelEntry* k = kernel_of(m, name);
  if (!k) return DAGRT_ENOTFOUND;
  if (nargs != (int32_t)k->kinds.size())
    return mfail(m, DAGRT_ESIG, "%s takes %zu arguments, got %d", name, k->kinds.size(), nargs);
  // distinct arrays with merged access (an array passed twice is one transfer)
  MArray* arr[kMaxArgs];
  bool rd[kMaxArgs], wr[kMaxArgs];
  int na = 0;
  double touched = 0.0;
  for (int i = 0; i < nargs; ++i) {
    const int32_t kd = k->kinds[i];
    if (!is_ptr(kd)) continue;
    MArray* a = get(m, args[i].array);
    if (!a) return mfail(m, DAGRT_ENOTFOUND, "%s arg %d: not a live multi-array", name, i);
    int j = 0;
    while (j < na && arr[j] != a) ++j;
    if (j == na) {
      arr[na] = a;
      rd[na] = wr[na] = false;
      touched += (double)a->bytes;
      ++na;
    }
    rd[j] = rd[j] || reads(kd);
    wr[j] = wr[j] || writes(kd);
  }
  const double exec_us = touched / (kHbmGBs * 1e3);
  int d = slot;
  double finish = 0.0;
  if (d < 0 && m->placement == DAGRT_PLACE_ROUND_ROBIN) d = (int)(m->rr++ % (uint64_t)n);
  if (d < 0) {  // earliest estimated finish: busy + migrations + own traffic
    for (int s = 0; s < n; ++s) {
      double t = m->slots[s].busy_us + exec_us;
      for (int j = 0; j < na; ++j) {
        if (!rd[j] || (arr[j]->valid & bit(s))) continue;
        int src;
        const double bw = source_of(m, arr[j], s, &src);
        if (src != -2) t += (double)arr[j]->bytes / (bw * 1e3);
      }
      if (d < 0 || t < finish) {
        d = s;
        finish = t;
      }
    }
  } else {
    finish = m->slots[d].busy_us + exec_us;
    for (int j = 0; j < na; ++j) {
      if (!rd[j] || (arr[j]->valid & bit(d))) continue;
      int src;
      const double bw = source_of(m, arr[j], d, &src);
      if (src != -2) finish += (double)arr[j]->bytes / (bw * 1e3);
    }
  }
  for (int j = 0; j < na; ++j) {
    if (rd[j]) {
      if (dagrt_status e = migrate(m, arr[j], d)) return e;
    } else if (dagrt_status e = ensure_replica(m, arr[j], d)) {
      return e;
    }
  }
  dagrt_arg local[kMaxArgs];
  for (int i = 0; i < nargs; ++i) {
    local[i] = args[i];
    if (is_ptr(k->kinds[i])) local[i].array = get(m, args[i].array)->rep[d].h;
  }
  if (dagrt_status e = set_dev(m, d)) return e;
  if (dagrt_status e = dagrt_launch(m->slots[d].ctx, k->h[d], grid, block, smem, local, nargs))
    return slot_fail(m, d, e, name);
  for (int j = 0; j < na; ++j)
    if (wr[j]) arr[j]->valid = bit(d);
  m->slots[d].busy_us = finish;
  m->st.launches++;
  m->st.per_slot[d]++;
  if (placed) *placed = d;
  return DAGRT_OK;
}

dagrt_status dagrt_multi_host_read(dagrt_multi m, dagrt_marray h, size_t off, size_t bytes, void* dst) {
  if (!m || (bytes && !dst)) return DAGRT_EINVAL;
  MArray* a = get(m, h);
  if (!a) return mfail(m, DAGRT_ENOTFOUND, "stale multi-array handle");
  if (off > a->bytes || bytes > a->bytes - off) return mfail(m, DAGRT_EINVAL, "range out of bounds");
  if ((a->valid & kHostBit) && a->host) {
    if (dst != a->host + off) std::memmove(dst, a->host + off, bytes);
    return DAGRT_OK;
  }
  int s = -1;
  if (a->valid & bit(a->home)) s = a->home;
  for (int t = 0; s < 0 && t < (int)m->slots.size(); ++t)
    if (a->valid & bit(t)) s = t;
  if (s < 0) return mfail(m, DAGRT_ESTATE, "multi-array has no current copy (never written)");
  if (dagrt_status e = set_dev(m, s)) return e;
  if (dagrt_status e = dagrt_host_read(m->slots[s].ctx, a->rep[s].h, off, bytes, dst))
    return slot_fail(m, s, e, "host read");
  if (a->host && dst == a->host && off == 0 && bytes == a->bytes) a->valid |= kHostBit;
  return DAGRT_OK;
}

dagrt_status dagrt_multi_host_write(dagrt_multi m, dagrt_marray h, size_t off, size_t bytes, const void* src) {
  if (!m || (bytes && !src)) return DAGRT_EINVAL;
  MArray* a = get(m, h);
  if (!a) return mfail(m, DAGRT_ENOTFOUND, "stale multi-array handle");
  if (off > a->bytes || bytes > a->bytes - off) return mfail(m, DAGRT_EINVAL, "range out of bounds");
  const bool whole = off == 0 && bytes == a->bytes;
  if (a->host) {
    // uploads still reading the mirror must finish before it changes
    for (int s = 0; s < (int)m->slots.size(); ++s)
      if ((a->uploading & bit(s)) && m->real && a->rep[s].up_ev) {
        cudaError_t e = cudaEventSynchronize((cudaEvent_t)a->rep[s].up_ev);
        if (e != cudaSuccess) return mfail(m, DAGRT_ECUDA, "upload wait: %s", cudaGetErrorName(e));
      }
    a->uploading = 0;
    if (!whole && !(a->valid & kHostBit) && a->valid)
      if (dagrt_status e = dagrt_multi_host_read(m, h, 0, a->bytes, a->host)) return e;
    if (src != a->host + off) std::memmove(a->host + off, src, bytes);
    a->valid = kHostBit;
    return DAGRT_OK;
  }
  const int home = a->home;
  if (!whole && a->valid)
    if (dagrt_status e = migrate(m, a, home)) return e;
  if (dagrt_status e = ensure_replica(m, a, home)) return e;
  if (dagrt_status e = set_dev(m, home)) return e;
  if (dagrt_status e = dagrt_host_write(m->slots[home].ctx, a->rep[home].h, off, bytes, src))
    return slot_fail(m, home, e, "host write");
  a->valid = bit(home);
  return DAGRT_OK;
}

dagrt_status dagrt_multi_sync(dagrt_multi m) {
  if (!m) return DAGRT_EINVAL;
  for (int s = 0; s < (int)m->slots.size(); ++s) {
    if (dagrt_status e = set_dev(m, s)) return e;
    if (dagrt_status e = dagrt_sync(m->slots[s].ctx)) return slot_fail(m, s, e, "sync");
    m->slots[s].busy_us = 0.0;
  }
  for (MArray& a : m->arrays) a.uploading = 0;
  return DAGRT_OK;
}

dagrt_status dagrt_multi_stats(dagrt_multi m, dagrt_multi_stats_t* out) {
  if (!m || !out) return DAGRT_EINVAL;
  *out = m->st;
  return DAGRT_OK;
}

}  // extern "C"
