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

// Persistent merge-path SpMV.  CTA b owns the contiguous tile range
// [b*per, (b+1)*per).  All its tile boundaries (up to 256 at a time) are
// located first by all 8 warps in parallel (32-ary searches).  Rows that
// cross tile boundaries INSIDE the CTA's range are carried from tile to tile
// in shared memory (no atomics, no fences); only the row crossing the CTA's
// start and the row crossing its end are finished across CTAs (spmv_deposit,
// slots indexed by CTA), so at most two deposits per CTA leave the per-tile
// critical path clean.
constexpr int kSpmvChunk = 256;

__global__ void __launch_bounds__(kSpmvThreads, 4) k_spmv(const int* __restrict__ row_ptr,
                                                       const int* __restrict__ col,
                                                       const float* __restrict__ x,
                                                       float* __restrict__ y, long long N) {
  __shared__ int s_bnd[kSpmvChunk + 1];
  // double-buffered staging (tile parity): the next tile's writes never race
  // with the previous tile's reads, so no barrier is needed before staging
  __shared__ float s_val_buf[2][kSpmvTile];
  __shared__ int s_rend_buf[2][kSpmvTile + 1];  // row ends relative to j0
  __shared__ float s_wsum[kSpmvThreads / 32];
  __shared__ int s_wflag[kSpmvThreads / 32];
  __shared__ int s_first_emitter;
  __shared__ float s_carry, s_head_val, s_cta_carry;
  const long long E = (long long)__ldg(row_ptr + N);
  const long long total = N + E;
  const long long ntiles = (total + kSpmvTile - 1) / kSpmvTile;
  const SpmvWs ws = spmv_ws(y, N, gridDim.x);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const long long per = (ntiles + gridDim.x - 1) / gridDim.x;
  const long long me = blockIdx.x;
  const long long tb0 = me * per;
  const long long te0 = min(ntiles, tb0 + per);
  if (tb0 >= te0) return;  // uniform per CTA
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  auto cta_of_diag = [&](long long d) { return (d / kSpmvTile) / per; };
  if (t == 0) s_cta_carry = 0.f;

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
    for (long long c = tb; c < te; ++c) {
      const long long d0 = c * kSpmvTile, d1 = min(total, d0 + kSpmvTile);
      const long long i0 = s_bnd[c - tb], i1 = s_bnd[c - tb + 1];
      const long long j0 = d0 - i0, j1 = d1 - i1;
      const int nn = (int)(j1 - j0), nr = (int)(i1 - i0);
      const int nre = (int)(min(i1, N - 1) - i0 + 1);
      // ---- stage: column indices, then gathers (8 loads in flight each), row ends
      int ci[kSpmvItems];
#pragma unroll
      for (int u = 0; u < kSpmvItems; ++u) {
        const int k = t + u * kSpmvThreads;
        ci[u] = k < nn ? ldg_hint(col + j0 + k, pol_stream) : 0;
      }
      int re[kSpmvItems + 1];
#pragma unroll
      for (int u = 0; u <= kSpmvItems; ++u) {
        const int k = t + u * kSpmvThreads;
        re[u] = k < nre ? ldg_hint(row_ptr + i0 + k + 1, pol_stream) : 0;
      }
      const int rp0 = __ldg(row_ptr + i0);
      float xv[kSpmvItems];
#pragma unroll
      for (int u = 0; u < kSpmvItems; ++u) {
        const int k = t + u * kSpmvThreads;
        xv[u] = k < nn ? ldg_hint(x + ci[u], pol_keep) : 0.f;
      }
      float* s_val = s_val_buf[c & 1];
      int* s_rend = s_rend_buf[c & 1];
      const int j0i = (int)j0;
#pragma unroll
      for (int u = 0; u < kSpmvItems; ++u) {
        const int k = t + u * kSpmvThreads;
        if (k < nn) s_val[k] = xv[u];
      }
#pragma unroll
      for (int u = 0; u <= kSpmvItems; ++u) {
        const int k = t + u * kSpmvThreads;
        if (k < nre) s_rend[k] = re[u] - j0i;
      }
      if (t == 0) s_first_emitter = kSpmvThreads;
      __syncthreads();  // (B)
      // ---- thread-local merge-path search and sequential consumption
      const int dl = min(t * kSpmvItems, nn + nr);
      int lo = max(0, dl - nn), hi = min(dl, nr);
      while (lo < hi) {
        const int p = (lo + hi) >> 1;
        if (s_rend[p] <= dl - p - 1) lo = p + 1;
        else hi = p;
      }
      int ri = lo, nj = dl - lo;
      const int de = min(dl + kSpmvItems, nn + nr);
      float sum = 0.f, first_val = 0.f;
      bool emitted = false;
      long long first_row = -1;
      for (int it = dl; it < de; ++it) {
        const bool row_end = (ri < nr) && (s_rend[ri] <= nj);
        if (row_end) {
          if (!emitted) {
            emitted = true;
            first_row = i0 + ri;
            first_val = sum;
          } else {
            stg_hint(y + i0 + ri, sum, pol_stream);
          }
          sum = 0.f;
          ++ri;
        } else {
          sum += s_val[nj];
          ++nj;
        }
      }
      // ---- segmented inclusive scan over threads (warp shuffles + one
      // fixed-order cross-warp step): s(t) = sum(t) + (emitted(t) ? 0 : s(t-1))
      float sc = sum;
      bool fl = emitted;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const float yv = __shfl_up_sync(0xffffffffu, sc, off);
        const bool f = __shfl_up_sync(0xffffffffu, fl, off);
        if (lane >= off && !fl) { sc += yv; fl = f; }
      }
      if (lane == 31) { s_wsum[warp] = sc; s_wflag[warp] = fl ? 1 : 0; }
      if (emitted) atomicMin(&s_first_emitter, t);
      __syncthreads();  // (C)
      float win = 0.f;
      for (int w = 0; w < warp; ++w) win = s_wflag[w] ? s_wsum[w] : win + s_wsum[w];
      const float s_incl = fl ? sc : sc + win;
      float incoming = __shfl_up_sync(0xffffffffu, s_incl, 1);  // s(t-1)
      if (lane == 0) incoming = win;
      const int fe = s_first_emitter;
      const bool cont = (long long)rp0 < j0;  // row i0 started before this tile
      const float carry_in = (cont && c > tb0) ? s_cta_carry : 0.f;
      const bool head_x = cont && cta_of_diag(i0 + rp0) < me;  // row i0 began in an earlier CTA
      if (emitted) {
        float v = first_val + incoming;
        if (t == fe && first_row == i0) {
          v += carry_in;
          if (head_x) s_head_val = v;
          else stg_hint(y + i0, v, pol_stream);
        } else {
          stg_hint(y + first_row, v, pol_stream);
        }
      }
      if (t == kSpmvThreads - 1) s_carry = s_incl;
      __syncthreads();  // (D)
      // running partial of the row crossing this tile's end (this CTA's share)
      const float new_carry = fe < kSpmvThreads ? s_carry : carry_in + s_carry;
      if (warp == 0) {
        if (fe < kSpmvThreads && head_x)
          spmv_deposit(ws, y, i0, cta_of_diag(i0 + rp0), me, me, s_head_val, true);
        if (c == te0 - 1 && i1 < N) {
          const long long rs = nr > 0 ? (long long)s_rend[nr - 1] + j0 : (long long)rp0;  // row_ptr[i1]
          const long long rend = (long long)s_rend[nr] + j0;                            // row_ptr[i1+1]
          const long long as = cta_of_diag(i1 + rs), ae = cta_of_diag(i1 + rend);
          if (ae > me && as <= me) spmv_deposit(ws, y, i1, as, ae, me, new_carry, false);
        }
      }
      if (t == 0) s_cta_carry = new_carry;  // read by the next tile after barrier (C)
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
