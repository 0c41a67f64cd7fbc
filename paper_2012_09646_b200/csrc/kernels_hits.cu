// HITS kernels for sm_100a (§V-B; Fig. 6;
// reading R-HITS in DESIGN.md): 0/1 CSR SpMV, L2 norm, divide.
//
// SpMV on a power-law graph (20M rows, average degree 3, hub rows with
// ~1.5M non-zeros).  The paper used LightSpMV [31] (Kepler-era dynamic row
// distribution).  On B200 the kernel is a deterministic MERGE-PATH SpMV:
// the merged sequence of N row-ends and E non-zeros is cut into equal tiles
// of 2048 items (one CTA each), so every CTA does the same work whatever
// the degree distribution:
//   1. two warps locate the tile's (row, nnz) start/end coordinates with a
//      32-ary merge-path search over row_ptr (5 probes instead of 25);
//   2. the CTA stages its gathered x[col] values and row ends in shared
//      memory with coalesced loads;
//   3. each thread consumes 8 items (binary-searched inside shared memory),
//      completed rows are written directly;
//   4. a fixed-shape block scan carries partial row sums across threads;
//   5. rows spanning several CTAs are finished by the LAST CTA to deposit
//      its partial (atomic arrival count per row), which adds the partials
//      in CTA order with a fixed warp tree -> bit-deterministic results,
//      no spinning, no float atomics.
// The output array y carries the cross-CTA workspace after its N floats
// (see spmv_ws_bytes), like the reduction outputs (kcommon.cuh RedOut).
#include "kcommon.cuh"

namespace dagrt {

constexpr int kSpmvThreads = 256;
constexpr int kSpmvItems = 8;
constexpr int kSpmvTile = kSpmvThreads * kSpmvItems;  // merge items per CTA

struct SpmvWs {
  float* part;    // [ncta] partial of the row crossing the CTA's end
  float* head;    // [ncta] partial of the row crossing the CTA's start (its end part)
  unsigned* cnt;  // [ncta] arrival counters, indexed by the row's first CTA
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
// Executed by warp 0 of the CTA.  `is_head` = this CTA is the row's last (ce).
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

// Tile geometry: tile c = diagonals [c*T, min((c+1)*T, N+E)), start
// coordinate (i0, j0), end (i1, j1).
struct SpmvTile {  // 32-bit: CSR offsets and row ids are int32 by construction
  int c, i0, j0, i1, j1;
};

// Per-thread staging registers for one tile (loaded ahead of use).
struct SpmvStage {
  float xv[kSpmvItems];     // gathered x values
  int re[kSpmvItems + 1];   // row ends
  int rp0;                  // row_ptr[i0]
};

__device__ __forceinline__ void stage_cols(const int* __restrict__ col, const SpmvTile& T,
                                           int (&ci)[kSpmvItems], uint64_t pol) {
  const int t = threadIdx.x;
  const int nn = T.j1 - T.j0;
#pragma unroll
  for (int u = 0; u < kSpmvItems; ++u) {
    const int k = t + u * kSpmvThreads;
    ci[u] = k < nn ? ldg_hint(col + T.j0 + k, pol) : 0;
  }
}

__device__ __forceinline__ void stage_rows(const int* __restrict__ row_ptr, long long N,
                                           const SpmvTile& T, SpmvStage& S, uint64_t pol) {
  const int t = threadIdx.x;
  const int nre = (int)(min((long long)T.i1, N - 1) - T.i0 + 1);
#pragma unroll
  for (int u = 0; u <= kSpmvItems; ++u) {
    const int k = t + u * kSpmvThreads;
    S.re[u] = k < nre ? ldg_hint(row_ptr + T.i0 + k + 1, pol) : 0;
  }
  S.rp0 = __ldg(row_ptr + T.i0);
}

__device__ __forceinline__ void stage_gather(const float* __restrict__ x, const SpmvTile& T,
                                             const int (&ci)[kSpmvItems], SpmvStage& S, uint64_t pol) {
  const int t = threadIdx.x;
  const int nn = T.j1 - T.j0;
#pragma unroll
  for (int u = 0; u < kSpmvItems; ++u) {
    const int k = t + u * kSpmvThreads;
    S.xv[u] = k < nn ? ldg_hint(x + ci[u], pol) : 0.f;
  }
}

// Process one staged tile (all threads): local merge search, sequential
// consumption, segmented scan, cross-CTA deposits.
__device__ __forceinline__ void spmv_process(float* __restrict__ y, long long N, const SpmvWs& ws,
                                             const SpmvTile& T, const float* s_val, const int* s_rend,
                                             int rp0) {
  const long long c = T.c, i0 = T.i0, j0 = T.j0, i1 = T.i1;
  const int t = threadIdx.x, warp = t >> 5;
  const int nn = (int)(T.j1 - T.j0), nr = (int)(T.i1 - T.i0);

  // thread-local merge-path search inside the tile (binary, shared memory)
  const int dl = min(t * kSpmvItems, nn + nr);
  int lo = max(0, dl - nn), hi = min(dl, nr);
  while (lo < hi) {
    const int p = (lo + hi) >> 1;
    if ((long long)s_rend[p] - j0 <= dl - p - 1) lo = p + 1;
    else hi = p;
  }
  int ri = lo, nj = dl - lo;  // local row index, local nnz index
  const int de = min(dl + kSpmvItems, nn + nr);
  float sum = 0.f;
  bool emitted = false;
  long long first_row = -1;
  float first_val = 0.f;
  for (int it = dl; it < de; ++it) {
    const bool row_end = (ri < nr) && ((long long)s_rend[ri] - j0 <= nj);
    if (row_end) {
      if (!emitted) {
        emitted = true;
        first_row = i0 + ri;
        first_val = sum;
      } else {
        y[i0 + ri] = sum;
      }
      sum = 0.f;
      ++ri;
    } else {
      sum += s_val[nj];
      ++nj;
    }
  }
  // segmented inclusive scan s(t) = sum(t) + (emitted(t) ? 0 : s(t-1)):
  // warp shuffles, then one cross-warp step through shared memory (fixed
  // combination order -> deterministic)
  const int lane = t & 31;
  float sc = sum;
  bool fl = emitted;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float yv = __shfl_up_sync(0xffffffffu, sc, off);
    const bool f = __shfl_up_sync(0xffffffffu, fl, off);
    if (lane >= off && !fl) { sc += yv; fl = f; }
  }
  __shared__ float s_wsum[kSpmvThreads / 32];
  __shared__ int s_wflag[kSpmvThreads / 32];
  __shared__ int s_first_emitter;
  __shared__ float s_carry;
  __shared__ float s_head_val;
  if (t == 0) s_first_emitter = kSpmvThreads;
  if (lane == 31) { s_wsum[warp] = sc; s_wflag[warp] = fl ? 1 : 0; }
  __syncthreads();
  if (emitted) atomicMin(&s_first_emitter, t);
  float win = 0.f;  // carry into this warp from warps 0 .. warp-1
  for (int w = 0; w < warp; ++w) win = s_wflag[w] ? s_wsum[w] : win + s_wsum[w];
  const float s_incl = fl ? sc : sc + win;
  float incoming = __shfl_up_sync(0xffffffffu, s_incl, 1);  // s(t-1)
  if (lane == 0) incoming = win;
  if (t == kSpmvThreads - 1) s_carry = s_incl;
  __syncthreads();
  const int fe = s_first_emitter;
  // row i0 started in an earlier tile iff row_ptr[i0] < j0
  const bool i0_spans = (long long)rp0 < j0;
  if (emitted) {
    const float v = first_val + incoming;
    if (t == fe && first_row == i0 && i0_spans) s_head_val = v;
    else y[first_row] = v;
  }
  __syncthreads();
  if (warp == 0) {
    // (a) row i0 crossing the tile start and ending here
    if (fe < kSpmvThreads && i0 < N && i0_spans) {
      const long long cs = (i0 + rp0) / kSpmvTile;
      spmv_deposit(ws, y, i0, cs, c, c, s_head_val, true);
    }
    // (b) carry row i1 crossing the tile end (its end item lies in a later tile)
    if (i1 < N) {
      const long long rs = nr > 0 ? (long long)s_rend[nr - 1] : (long long)rp0;  // row_ptr[i1]
      const long long re = (long long)s_rend[nr];                               // row_ptr[i1+1]
      const long long cs = (i1 + rs) / kSpmvTile, ce = (i1 + re) / kSpmvTile;
      if (ce > c && cs <= c) spmv_deposit(ws, y, i1, cs, ce, c, s_carry, false);
    }
  }
}

// Persistent merge-path SpMV: each CTA owns a contiguous range of tiles.  All
// its tile boundaries (up to 256 at a time) are located first, by all 8
// warps in parallel (32-ary searches).  Tile staging is software-pipelined
// two deep in registers: while tile c is processed from shared memory, the
// gathers of tile c+1 and the column indices / row ends of tile c+2 are in
// flight, so the dependent col -> x latency chain is off the critical path.
constexpr int kSpmvChunk = 256;

__global__ void __launch_bounds__(kSpmvThreads, 3) k_spmv(const int* __restrict__ row_ptr,
                                                       const int* __restrict__ col,
                                                       const float* __restrict__ x,
                                                       float* __restrict__ y, long long N) {
  __shared__ int s_bnd[kSpmvChunk + 1];
  __shared__ float s_val[kSpmvTile];
  __shared__ int s_rend[kSpmvTile + 1];
  __shared__ int s_rp0;
  const long long E = (long long)__ldg(row_ptr + N);
  const long long total = N + E;
  const long long ntiles = (total + kSpmvTile - 1) / kSpmvTile;
  const SpmvWs ws = spmv_ws(y, N, ntiles);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const long long per = (ntiles + gridDim.x - 1) / gridDim.x;
  const long long tb0 = (long long)blockIdx.x * per;
  const long long te0 = min(ntiles, tb0 + per);
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  for (long long tb = tb0; tb < te0; tb += kSpmvChunk) {
    const long long te = min(te0, tb + kSpmvChunk);
    const int nb = (int)(te - tb) + 1;
    __syncthreads();  // s_bnd of the previous chunk consumed
    for (int b = warp; b < nb; b += kSpmvThreads / 32) {
      const long long d = min(total, (tb + b) * (long long)kSpmvTile);
      const long long i = warp_merge_search(row_ptr, N, E, d);
      if (lane == 0) s_bnd[b] = (int)i;
    }
    __syncthreads();
    auto tile_of = [&](long long c) {
      SpmvTile T;
      T.c = (int)c;
      const long long d0 = c * kSpmvTile, d1 = min(total, d0 + kSpmvTile);
      T.i0 = s_bnd[c - tb];
      T.i1 = s_bnd[c - tb + 1];
      T.j0 = (int)(d0 - T.i0);
      T.j1 = (int)(d1 - T.i1);
      return T;
    };
    // prologue: tile tb fully staged, column indices of tile tb+1 in flight
    SpmvStage cur, nxt;
    int ci[kSpmvItems];
    SpmvTile Tc = tile_of(tb);
    stage_cols(col, Tc, ci, pol_stream);
    stage_rows(row_ptr, N, Tc, cur, pol_stream);
    stage_gather(x, Tc, ci, cur, pol_keep);
    SpmvTile Tn = Tc;
    if (tb + 1 < te) {
      Tn = tile_of(tb + 1);
      stage_cols(col, Tn, ci, pol_stream);
    }
    for (long long c = tb; c < te; ++c) {
      const int nn = Tc.j1 - Tc.j0;
      const int nre = (int)(min((long long)Tc.i1, N - 1) - Tc.i0 + 1);
      __syncthreads();  // previous tile's readers of s_val / s_rend are done
#pragma unroll
      for (int u = 0; u < kSpmvItems; ++u) {
        const int k = t + u * kSpmvThreads;
        if (k < nn) s_val[k] = cur.xv[u];
      }
#pragma unroll
      for (int u = 0; u <= kSpmvItems; ++u) {
        const int k = t + u * kSpmvThreads;
        if (k < nre) s_rend[k] = cur.re[u];
      }
      if (t == 0) s_rp0 = cur.rp0;
      __syncthreads();
      const int rp0 = s_rp0;
      // pipeline: gathers + row ends of tile c+1 (its column indices arrived
      // during tile c-1), column indices of tile c+2
      SpmvTile T2 = Tn;
      if (c + 1 < te) {
        stage_gather(x, Tn, ci, nxt, pol_keep);
        stage_rows(row_ptr, N, Tn, nxt, pol_stream);
      }
      if (c + 2 < te) {
        T2 = tile_of(c + 2);
        stage_cols(col, T2, ci, pol_stream);
      }
      spmv_process(y, N, ws, Tc, s_val, s_rend, rp0);
      cur = nxt;
      Tc = Tn;
      Tn = T2;
    }
  }
}

// SUM node read as the L2 norm: n = sqrt(sum v^2), fp64 accumulation.
__global__ void __launch_bounds__(256) k_l2norm(const float* __restrict__ v, RedOut* out,
                                                long long n) {
  __shared__ double sh[32];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long long done = 0;
  if (aligned16(v)) {
    const long long n4 = n >> 2;
    const float4* v4 = reinterpret_cast<const float4*>(v);
    for (long long i = tid; i < n4; i += nth) {
      float4 a = ldg_stream(v4 + i);
      acc += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) acc += (double)v[i] * v[i];
  double blk = block_reduce(acc, OpAdd(), sh);
  double total;
  if (grid_finish(out, blk, OpAdd(), 0.0, &total, sh) && threadIdx.x == 0)
    out->result = (float)sqrt(total);
}

// DIV node: out = v / ||v|| (zeros if the norm is 0).
__global__ void __launch_bounds__(256) k_divide(const float* __restrict__ v,
                                                const RedOut* __restrict__ nrm,
                                                float* __restrict__ out, long long n) {
  const float s = nrm->result;
  const float is = s > 0.f ? 1.f / s : 0.f;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(v) && aligned16(out)) {
    const long long n4 = n >> 2;
    for (long long i = tid; i < n4; i += nth) {
      float4 a = ldg_stream(reinterpret_cast<const float4*>(v) + i);
      a.x *= is; a.y *= is; a.z *= is; a.w *= is;
      reinterpret_cast<float4*>(out)[i] = a;
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) out[i] = v[i] * is;
}

static const Builtin kHits[] = {
    {"spmv", (const void*)k_spmv, "const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE},
    {"l2norm", (const void*)k_l2norm, "const ptr, out ptr, sint64", KF_NONE},
    {"divide", (const void*)k_divide, "const ptr, const ptr, out ptr, sint64", KF_NONE},
};
DAGRT_REGISTER_BUILTINS(kHits);

}  // namespace dagrt
