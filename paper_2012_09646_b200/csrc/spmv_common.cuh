// SpMV building blocks shared by the product kernel (kernels_hits.cu) and
// its experimental variants (exp/spmv_variants.cu): the cross-warp
// workspace and deposit protocols that make rows spanning several warps
// bit-reproducible, and the streamed column loads of the non-zero split.
#pragma once
#include "kcommon.cuh"

namespace dagrt {

constexpr int kSpmvThreads = 256;
constexpr int kSpmvWarps = kSpmvThreads / 32;
constexpr int kSpmvItems = 8;                 // merge items per lane
constexpr int kSpmvTile = 32 * kSpmvItems;    // merge items per warp tile

// Cross-warp workspace, one slot per participant (global warp of the grid).
struct SpmvWs {
  float* part;    // [G] share of the row crossing the warp range's end
  float* head;    // [G] share of the row crossing the range's start (its end part)
  unsigned* cnt;  // [G] arrival counters, indexed by the row's first participant
};

__device__ __forceinline__ SpmvWs spmv_ws(float* y, long long n, long long ncta) {
  uintptr_t base = (uintptr_t)(y + n);
  base = (base + 15) & ~(uintptr_t)15;
  SpmvWs w;
  w.part = reinterpret_cast<float*>(base);
  w.head = w.part + ncta;
  w.cnt = reinterpret_cast<unsigned*>(w.head + ncta);
  return w;
}

// Merge-path coordinate of diagonal d: rows consumed i (row-end items) and
// non-zeros consumed j = d - i.  Row-end i precedes nnz j iff row_ptr[i+1] <= j.
// Executed by one full warp; 32-ary search.
__device__ __forceinline__ long long warp_merge_search(const int* __restrict__ row_ptr, long long N,
                                                       long long E, long long d) {
  const int lane = threadIdx.x & 31;
  long long lo = d - E > 0 ? d - E : 0;
  long long hi = d < N ? d : N;
  while (hi - lo > 32) {
    const long long step = (hi - lo + 31) / 32;
    const long long p = lo + lane * step;
    bool pred = false;
    if (p < hi) pred = (long long)__ldg(row_ptr + p + 1) <= d - p - 1;
    const unsigned b = __ballot_sync(0xffffffffu, pred);
    const int cnt = __popc(b);  // predicate holds on a prefix of the probes
    const long long nlo = cnt > 0 ? lo + (long long)(cnt - 1) * step + 1 : lo;
    const long long nhi = min(hi, lo + (long long)cnt * step);
    lo = nlo;
    hi = nhi;
  }
  const long long p = lo + lane;
  bool pred = false;
  if (p < hi) pred = (long long)__ldg(row_ptr + p + 1) <= d - p - 1;
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  return lo + __popc(b);
}

// Sum v[first..last] (fixed order: lane-strided partial sums, fixed tree) by one warp.
__device__ __forceinline__ float warp_ordered_sum(const volatile float* v, long long first,
                                                  long long last) {
  const int lane = threadIdx.x & 31;
  float s = 0.f;
  for (long long k = first + lane; k <= last; k += 32) s += v[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Deposit `val` for row r (spanning CTAs cs..ce) and finish the row if last.
// Executed by one whole warp.  `is_head` = this participant holds the row's end (ce).
__device__ __forceinline__ void spmv_deposit(const SpmvWs& ws, float* y, long long r, long long cs,
                                             long long ce, long long c, float val, bool is_head) {
  const int lane = threadIdx.x & 31;
  unsigned old = 0;
  if (lane == 0) {
    if (is_head) ws.head[c] = val;
    else ws.part[c] = val;
    __threadfence();
    old = atomicAdd(ws.cnt + cs, 1u);
  }
  old = __shfl_sync(0xffffffffu, old, 0);
  if (old == (unsigned)(ce - cs)) {  // last of the (ce - cs + 1) participants
    __threadfence();
    float s = warp_ordered_sum(ws.part, cs, ce - 1);
    if (lane == 0) {
      s += ((volatile float*)ws.head)[ce];
      y[r] = s;
      ws.cnt[cs] = 0;  // reusable by the next launch
    }
  }
}

// Single-thread deposit protocol (spmv_nz): participant c puts its share of
// a row spanning warps cs..ce (the end participant into head[], the others
// into part[]); the last to arrive at cnt[cs] adds them in warp order.
__device__ __forceinline__ void spmv_ws_put(const SpmvWs& ws, long long c, float val, bool is_end) {
  if (is_end) ws.head[c] = val;
  else ws.part[c] = val;
}
__device__ __forceinline__ bool spmv_ws_arrive(const SpmvWs& ws, long long cs, long long ce) {
  __threadfence();
  const unsigned old = atomicAdd(ws.cnt + cs, 1u);
  if (old != (unsigned)(ce - cs)) return false;
  __threadfence();
  ws.cnt[cs] = 0;  // reusable by the next launch
  return true;
}
__device__ __forceinline__ float spmv_ws_sum(const SpmvWs& ws, long long cs, long long ce) {
  float s = 0.f;
  const volatile float* p = ws.part;
  for (long long c = cs; c < ce; ++c) s += p[c];
  return s + ((volatile float*)ws.head)[ce];
}

constexpr int kNzChunk = 128;  // non-zeros per warp chunk (4 per lane)
constexpr int kNzHeader = 16;  // plan header ints

__device__ __forceinline__ int4 ld_cols_stream(const int* p, uint64_t pol) {
  int4 c;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(p), "l"(pol));
  return c;
}

// One chunk's streamed inputs for one lane: its 4 column indices, and the
// chunk's 4 row-start flag words (the same 16 bytes for every lane: one
// broadcast load).  The flag words are used only when the chunk is reduced,
// so their latency is covered by the pipeline like the columns'.
struct NzIn {
  int c[4];
  uint4 fw;
};

__device__ __forceinline__ void nz_gather(const NzIn& in, const float* __restrict__ x, float (&v)[4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) v[u] = in.c[u] >= 0 ? __ldg(x + in.c[u]) : 0.f;
}

// ---------------------------------------------------------------------------
// "spmv" (product, round 2): the non-zero split of spmv_nz (exp/spmv_variants.cu,
// whose notes describe the chunk pipeline, the segmented warp scan and the
// cross-warp deposits this kernel shares) with EVERY row padded
// to at least one item -- each empty row gets one column index -1 (value 0)
// when the graph is registered (spmv_pad_plan(), programs/hits_dl.py).  Then
// ordinals ARE row ids: completed rows are written to consecutive addresses
// with no row-id loads and no zero-filling of skipped rows (the profile of
// spmv_nz put its top stalls on exactly those: the row-id loads and the
// divergent gap loops), at the cost of 9M more 4-byte column indices on the
// HBM-cheap coalesced stream.  Plan (int32): [header(16) | rp2(N+1) |
// rbase(nc+1) | flags(4 nc + 4 words) | ci2(E2)], rp2 the padded row
// pointers (used only for rows crossing warp ranges), E2 = E + #empty rows.
constexpr int kPadMagic = 0x50414430;  // "PAD0"

struct PadPlan {
  int nc, n, e2;
  const int* rp2;
  const int* rbase;
  const unsigned* flags;
  const int* ci2;
};

__device__ __forceinline__ PadPlan pad_plan(const int* plan) {
  if (__ldg(plan) != kPadMagic || __ldg(plan + 3) != kNzChunk) __trap();  // built for another kernel
  PadPlan P;
  P.nc = __ldg(plan + 1);
  P.n = __ldg(plan + 2);
  P.rp2 = plan + __ldg(plan + 4);
  P.rbase = plan + __ldg(plan + 5);
  P.flags = reinterpret_cast<const unsigned*>(plan + __ldg(plan + 6));
  P.ci2 = plan + __ldg(plan + 7);
  P.e2 = __ldg(plan + 8);
  return P;
}

__device__ __forceinline__ NzIn pad_load(const PadPlan& P, int chunk, int lane, uint64_t pol) {
  NzIn in;
  const int k = chunk * kNzChunk + 4 * lane;
  if (k + 3 < P.e2) {
    const int4 q = ld_cols_stream(P.ci2 + k, pol);
    in.c[0] = q.x; in.c[1] = q.y; in.c[2] = q.z; in.c[3] = q.w;
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) in.c[u] = k + u < P.e2 ? __ldg(P.ci2 + k + u) : -1;
  }
  in.fw = __ldg(reinterpret_cast<const uint4*>(P.flags) + chunk);
  return in;
}

template <bool HINTS>
__device__ __forceinline__ void nz_gather_h(const NzIn& in, const float* __restrict__ x, float (&v)[4], uint64_t keep) {
  if (!HINTS) {
    nz_gather(in, x, v);
    return;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) v[u] = in.c[u] >= 0 ? ldg_hint(x + in.c[u], keep) : 0.f;
}

// The padded non-zero split (k_spmv_pad, kernels_hits.cu).  HINTS: the
// gathers carry an L2 evict_last policy and the y stores evict_first, so the
// streamed output does not push the gathered vector out of L2 (an
// experimental form, exp/spmv_variants.cu).
template <bool HINTS>
__device__ __forceinline__ void spmv_pad_body(const int* __restrict__ plan, const float* __restrict__ x,
                                              float* __restrict__ y, long long N_) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const PadPlan P = pad_plan(plan);
  if ((long long)P.n != N_ || P.n == 0) return;
  const int G = (int)gridDim.x * (blockDim.x >> 5);
  const int g = (int)blockIdx.x * (blockDim.x >> 5) + warp;
  const int per = (P.nc + G - 1) / G;
  const int cb = g * per, ce = min(P.nc, cb + per);
  if (cb >= ce) return;  // warp-uniform; the kernel has no CTA barriers
  const SpmvWs ws = spmv_ws(y, N_, G);
  const uint64_t pol = l2_policy_evict_first();
  const uint64_t keep = HINTS ? l2_policy_evict_last() : 0;
  auto store = [&](int i, float v) {
    if (HINTS)
      asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(y + i), "f"(v), "l"(pol) : "memory");
    else
      y[i] = v;
  };
  auto warp_of_item = [&](int k) { return (k / kNzChunk) / per; };
  const int wsel = lane >> 3, bsh = 4 * (lane & 7);
  const unsigned lanes_below = (1u << lane) - 1u;

  const int k0w = cb * kNzChunk;
  const bool start0 = (__ldg(P.flags + (k0w >> 5)) >> (k0w & 31)) & 1u;
  int R0 = __ldg(P.rbase + cb);  // row open at the current chunk's start
  bool head_pending = !start0;   // ... which began in an earlier warp's range
  float carry = 0.f;

  NzIn cur = pad_load(P, cb, lane, pol);
  NzIn nxt = cur;
  if (cb + 1 < ce) nxt = pad_load(P, cb + 1, lane, pol);
  float v[4];
  nz_gather_h<HINTS>(cur, x, v, keep);
  for (int c = cb; c < ce; ++c) {
    uint4 fw = cur.fw;
    if (c == cb) fw.x &= ~1u;  // the range's first item: handled by start0/head_pending
    const unsigned mine = wsel == 0 ? fw.x : (wsel == 1 ? fw.y : (wsel == 2 ? fw.z : fw.w));
    const unsigned fl = (mine >> bsh) & 0xFu;
    const int nst = __popc(fl);
    const int before = (wsel > 0 ? __popc(fw.x) : 0) + (wsel > 1 ? __popc(fw.y) : 0) +
                       (wsel > 2 ? __popc(fw.z) : 0) + __popc(mine & ((1u << bsh) - 1u));
    const int total = __popc(fw.x) + __popc(fw.y) + __popc(fw.z) + __popc(fw.w);
    const int o = R0 + before;  // row open entering the lane; ends at its first start
    float vn[4] = {0.f, 0.f, 0.f, 0.f};
    if (c + 1 < ce) {
      nz_gather_h<HINTS>(nxt, x, vn, keep);
      cur = nxt;
      if (c + 2 < ce) nxt = pad_load(P, c + 2, lane, pol);
    }
    float run = 0.f, head = 0.f;
    bool seen = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if ((fl >> u) & 1u) {
        if (!seen) head = run;
        seen = true;
        run = 0.f;
      }
      run += v[u];
    }
    if (!seen) head = run;
    const unsigned m = __ballot_sync(0xffffffffu, nst != 0);
    float sv = nst ? run : head;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float tv = __shfl_up_sync(0xffffffffu, sv, off);
      const unsigned win = lane >= off ? (m >> (lane - off + 1)) & ((1u << off) - 1u) : 1u;
      if (win == 0u) sv += tv;
    }
    float cin = __shfl_up_sync(0xffffffffu, sv, 1);
    if (lane == 0) cin = 0.f;
    if ((m & lanes_below) == 0u) cin += carry;
    if (nst) {
      const float val = cin + head;
      if (head_pending && before == 0) {
        const int cs = warp_of_item(__ldg(P.rp2 + o));
        spmv_ws_put(ws, g, val, true);
        if (spmv_ws_arrive(ws, cs, g)) y[o] = spmv_ws_sum(ws, cs, g);
      } else {
        store(o, val);
      }
      int j = 1;
      float r2 = 0.f;
      bool in = false;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if ((fl >> u) & 1u) {
          if (in) store(o + j++, r2);
          in = true;
          r2 = 0.f;
        }
        r2 += v[u];
      }
    }
    const float tail_all = __shfl_sync(0xffffffffu, sv, 31);
    carry = m ? tail_all : carry + tail_all;
    if (m) head_pending = false;
    R0 += total;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = vn[u];
  }
  // the row open at the range end
  if (lane == 0) {
    const int ke = ce * kNzChunk;
    const bool ends_here = ke >= P.e2 || ((__ldg(P.flags + (ke >> 5)) >> (ke & 31)) & 1u);
    if (ends_here) {
      if (head_pending) {  // spans the whole range, ends at its end
        const int cs = warp_of_item(__ldg(P.rp2 + R0));
        spmv_ws_put(ws, g, carry, true);
        if (spmv_ws_arrive(ws, cs, g)) y[R0] = spmv_ws_sum(ws, cs, g);
      } else {
        store(R0, carry);
      }
    } else {
      const int cs = warp_of_item(__ldg(P.rp2 + R0));
      const int cend = warp_of_item(__ldg(P.rp2 + R0 + 1) - 1);
      spmv_ws_put(ws, g, carry, false);
      if (spmv_ws_arrive(ws, cs, cend)) y[R0] = spmv_ws_sum(ws, cs, cend);
    }
  }
}

// ---------------------------------------------------------------------------
// spmv_pad2 (the product "spmv" since round 2's end): the padded non-zero split with the segmented warp scan
// taken only where it is needed.  ncu on the product (profiles/r2_ncu_*): the
// top stall is short_scoreboard (shuffle latency of the 5-step scan run on
// every 128-item chunk).  Per chunk, m = lanes holding a row start:
//   m == 0   (the chunk lies inside one row -- the hubs hold half of the
//            non-zeros): each lane adds its 4 items to a per-lane partial;
//            no shuffle at all; the partials are reduced (xor tree) once,
//            when the row ends;
//   m == all (every lane starts a row: rows span at most two lanes): a lane's
//            first row is the previous lane's tail plus its head -- one
//            shuffle up, one broadcast for the carry;
//   else     the segmented scan as in the product.
// Same rows, same deposits; fp32 sums in a different (fixed) order.
//
// HUB: the gathers of the hot head of x come from shared memory.  On the
// degree-ordered HITS graph (vertices relabelled by descending degree when the
// graph is registered, programs/hits_dl.py degree_order) the first H entries
// of x are the hubs that most non-zeros point at; each CTA stages x[0, H) once
// (H = dynamic shared memory / 4, a launch parameter) and every gather with a
// column below H is a shared-memory load instead of an L1/L2 request -- the
// request rate of the random gathers is this kernel's bound (tools/spmv_lab.py).
// The values are the same, so the sums are bit-identical to HUB = false.
__device__ __forceinline__ int hub_stage(const float* __restrict__ x, int n, float* hub) {
  unsigned dyn;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  int H = min((int)(dyn >> 2), n) & ~3;
  if (!aligned16(x)) H = 0;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4* h4 = reinterpret_cast<float4*>(hub);
  for (int i = threadIdx.x; i < (H >> 2); i += blockDim.x) h4[i] = __ldg(x4 + i);
  __syncthreads();
  return H;
}
__device__ __forceinline__ void nz_gather_hub(const NzIn& in, const float* __restrict__ x, const float* hub,
                                              int H, float (&v)[4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = in.c[u];
    v[u] = (unsigned)c < (unsigned)H ? hub[c] : (c >= 0 ? __ldg(x + c) : 0.f);
  }
}

template <int MINB, bool HUB = false>
__device__ __forceinline__ void spmv_pad2_body(const int* __restrict__ plan, const float* __restrict__ x,
                                               float* __restrict__ y, long long N_) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const PadPlan P = pad_plan(plan);
  if ((long long)P.n != N_ || P.n == 0) return;
  extern __shared__ __align__(16) float hub_sm[];
  const int H = HUB ? hub_stage(x, P.n, hub_sm) : 0;
  auto gather = [&](const NzIn& in, float (&vv)[4]) {
    if (HUB) nz_gather_hub(in, x, hub_sm, H, vv);
    else nz_gather(in, x, vv);
  };
  const int G = (int)gridDim.x * (blockDim.x >> 5);
  const int g = (int)blockIdx.x * (blockDim.x >> 5) + warp;
  const int per = (P.nc + G - 1) / G;
  const int cb = g * per, ce = min(P.nc, cb + per);
  if (cb >= ce) return;
  const SpmvWs ws = spmv_ws(y, N_, G);
  const uint64_t pol = l2_policy_evict_first();
  auto warp_of_item = [&](int k) { return (k / kNzChunk) / per; };
  const int wsel = lane >> 3, bsh = 4 * (lane & 7);
  const unsigned lanes_below = (1u << lane) - 1u;

  const int k0w = cb * kNzChunk;
  const bool start0 = (__ldg(P.flags + (k0w >> 5)) >> (k0w & 31)) & 1u;
  int R0 = __ldg(P.rbase + cb);
  bool head_pending = !start0;
  float carry = 0.f;       // warp-uniform part of the open row's partial sum
  float carry_lane = 0.f;  // per-lane part, from chunks without a row start
  bool dist = false;       // carry_lane is non-empty somewhere (warp-uniform)

  NzIn cur = pad_load(P, cb, lane, pol);
  NzIn nxt = cur;
  if (cb + 1 < ce) nxt = pad_load(P, cb + 1, lane, pol);
  float v[4];
  gather(cur, v);
  for (int c = cb; c < ce; ++c) {
    uint4 fw = cur.fw;
    if (c == cb) fw.x &= ~1u;
    const unsigned mine = wsel == 0 ? fw.x : (wsel == 1 ? fw.y : (wsel == 2 ? fw.z : fw.w));
    const unsigned fl = (mine >> bsh) & 0xFu;
    const int nst = __popc(fl);
    float vn[4] = {0.f, 0.f, 0.f, 0.f};
    if (c + 1 < ce) {
      gather(nxt, vn);
      cur = nxt;
      if (c + 2 < ce) nxt = pad_load(P, c + 2, lane, pol);
    }
    const unsigned m = __ballot_sync(0xffffffffu, nst != 0);
    if (m == 0u) {  // inside one row
      carry_lane += (v[0] + v[1]) + (v[2] + v[3]);
      dist = true;
    } else {
      if (dist) {
        float t = carry_lane;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        carry += t;
        carry_lane = 0.f;
        dist = false;
      }
      const int before = (wsel > 0 ? __popc(fw.x) : 0) + (wsel > 1 ? __popc(fw.y) : 0) +
                         (wsel > 2 ? __popc(fw.z) : 0) + __popc(mine & ((1u << bsh) - 1u));
      const int total = __popc(fw.x) + __popc(fw.y) + __popc(fw.z) + __popc(fw.w);
      const int o = R0 + before;
      float run = 0.f, head = 0.f;
      bool seen = false;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if ((fl >> u) & 1u) {
          if (!seen) head = run;
          seen = true;
          run = 0.f;
        }
        run += v[u];
      }
      if (!seen) head = run;
      float cin, tail_all;
      if (m == 0xffffffffu) {  // rows span at most two lanes
        cin = __shfl_up_sync(0xffffffffu, run, 1);
        if (lane == 0) cin = carry;
        tail_all = __shfl_sync(0xffffffffu, run, 31);
      } else {
        float sv = nst ? run : head;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float tv = __shfl_up_sync(0xffffffffu, sv, off);
          const unsigned win = lane >= off ? (m >> (lane - off + 1)) & ((1u << off) - 1u) : 1u;
          if (win == 0u) sv += tv;
        }
        cin = __shfl_up_sync(0xffffffffu, sv, 1);
        if (lane == 0) cin = 0.f;
        if ((m & lanes_below) == 0u) cin += carry;
        tail_all = __shfl_sync(0xffffffffu, sv, 31);
      }
      if (nst) {
        const float val = cin + head;
        if (head_pending && before == 0) {
          const int cs = warp_of_item(__ldg(P.rp2 + o));
          spmv_ws_put(ws, g, val, true);
          if (spmv_ws_arrive(ws, cs, g)) y[o] = spmv_ws_sum(ws, cs, g);
        } else {
          y[o] = val;
        }
        int j = 1;
        float r2 = 0.f;
        bool in = false;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if ((fl >> u) & 1u) {
            if (in) y[o + j++] = r2;
            in = true;
            r2 = 0.f;
          }
          r2 += v[u];
        }
      }
      carry = tail_all;
      head_pending = false;
      R0 += total;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = vn[u];
  }
  if (dist) {
    float t = carry_lane;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    carry += t;
  }
  if (lane == 0) {
    const int ke = ce * kNzChunk;
    const bool ends_here = ke >= P.e2 || ((__ldg(P.flags + (ke >> 5)) >> (ke & 31)) & 1u);
    if (ends_here) {
      if (head_pending) {
        const int cs = warp_of_item(__ldg(P.rp2 + R0));
        spmv_ws_put(ws, g, carry, true);
        if (spmv_ws_arrive(ws, cs, g)) y[R0] = spmv_ws_sum(ws, cs, g);
      } else {
        y[R0] = carry;
      }
    } else {
      const int cs = warp_of_item(__ldg(P.rp2 + R0));
      const int cend = warp_of_item(__ldg(P.rp2 + R0 + 1) - 1);
      spmv_ws_put(ws, g, carry, false);
      if (spmv_ws_arrive(ws, cs, cend)) y[R0] = spmv_ws_sum(ws, cs, cend);
    }
  }
}
// launch contract of the plan-driven kernels (builtin.h LaunchCheck)
static inline const char* v_spmv_plan_kernel(const LaunchCheck& L) {  // row_ptr, col, plan, x, y, N
  const int64_t N = L.i(5);
  if (N < 0 || N >= (1ll << 31)) return "need 0 <= N < 2^31";
  if (!fits(L, 0, 4ull * (N + 1))) return "row_ptr needs 4 (N + 1) bytes";
  if (!fits(L, 2, 4ull * kNzHeader)) return "plan smaller than its header";
  if (!fits(L, 3, 4ull * N)) return "x needs 4 N bytes";
  if (L.block[0] % 32 || L.block[1] != 1 || L.block[2] != 1 || L.grid[1] != 1 || L.grid[2] != 1)
    return "1-D launch, block a multiple of 32";
  // y carries the cross-warp workspace: 16-byte aligned after N floats, 3 words per warp
  if (!fits(L, 4, 4ull * N + 16 + 12ull * (L.block[0] / 32) * L.grid[0]))
    return "y needs 4 N + 16 + 12 (warps of the grid) bytes";
  return nullptr;
}

}  // namespace dagrt
