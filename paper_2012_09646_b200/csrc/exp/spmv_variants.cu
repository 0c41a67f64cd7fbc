// Experimental SpMV variants (libdagrt_exp.so; see exp_common.cuh), each
// exact and tested against the product kernel and the oracle:
//  * spmv_merge (+ spmv_sync / _x0s1 / _x1s1 / _as1 L2-policy and
//    pipelining variants): the round-1 merge-path kernel, 364 us on the HITS
//    graph;
//  * spmv_plan / spmv_plan_h: split by row class, 375-490 us;
//  * spmv_nz: the non-zero split without row padding (row ids from a
//    non-empty-row list); the product pads empty rows instead.
#include "../spmv_common.cuh"
#include "exp_common.cuh"
#include "../bs_math.cuh"  // bs_mbar_init / bs_mbar_wait

namespace dagrt {

// Persistent merge-path SpMV with WARP tiles.  Global warp g of G owns the
// contiguous merge range of tiles [g*per, (g+1)*per), each tile 256 items
// (8 per lane).  Warps never wait for each other (no CTA barriers): a warp
// finds its start with one 32-ary search, then walks its tiles with the row
// ends and column indices of tile c+1 in flight while tile c is gathered and
// reduced.  Per tile:
//   1. nr = rows ending in the tile = #{p : pos(p) < L}, pos(p) = p +
//      row_ptr[i0+p+1] - j0 the merge index of row end p (ballot counts;
//      the predicate holds on a prefix, so no search is needed);
//   2. gathers x[col] for the tile's nn = L - nr non-zeros;
//   3. row ends are marked in a byte map; each lane reads the 8 marks of its
//      items, an exclusive warp scan of the mark counts gives its first row
//      and non-zero, and it reduces its items sequentially;
//   4. a segmented warp scan carries partial rows across lanes, the warp's
//      running carry across tiles; completed rows are written to y[i0..i1)
//      from shared memory, coalesced.
// Rows spanning several warp ranges are finished by spmv_deposit.
// L2 policy variants (tools/spmv_variants.py): XP for the x gathers (0 default,
// 1 evict-last), SP for the streamed CSR arrays and y (0 default, 1 evict-first,
// 2 evict-first and no L1 allocation).
template <int XP, int SP>
__device__ __forceinline__ int spmv_ld_stream(const int* p, uint64_t pol) {
  if (SP == 0) return __ldg(p);
  if (SP == 1) return ldg_hint(p, pol);
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
template <int XP>
__device__ __forceinline__ float spmv_ld_x(const float* p, uint64_t pol) {
  return XP == 1 ? ldg_hint(p, pol) : __ldg(p);
}

template <int XP, int SP>
__device__ __forceinline__ void spmv_body(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                          const float* __restrict__ x, float* __restrict__ y,
                                          long long N_) {
  __shared__ float s_val_all[kSpmvWarps][kSpmvTile];
  __shared__ float s_y_all[kSpmvWarps][kSpmvTile];
  __shared__ __align__(16) unsigned char s_mark_all[kSpmvWarps][kSpmvTile];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* s_val = s_val_all[warp];
  float* s_y = s_y_all[warp];
  unsigned char* s_mark = s_mark_all[warp];
  const long long E_ = (long long)__ldg(row_ptr + N_);
  if (N_ + E_ + kSpmvTile >= (1ll << 31)) __trap();  // merge coordinates are 32-bit (documented limit)
  const int N = (int)N_, E = (int)E_, total = N + E;
  const int ntiles = (total + kSpmvTile - 1) / kSpmvTile;
  const int G = (int)gridDim.x * kSpmvWarps;
  const int g = (int)blockIdx.x * kSpmvWarps + warp;
  const int per = (ntiles + G - 1) / G;
  const int tb = g * per, te = min(ntiles, tb + per);
  if (tb >= te) return;  // warp-uniform; the kernel has no CTA barriers
  const SpmvWs ws = spmv_ws(y, N_, G);
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  auto warp_of_diag = [&](long long d) { return (d / kSpmvTile) / per; };

  int i0 = (int)warp_merge_search(row_ptr, N_, E_, (long long)tb * kSpmvTile);
  int j0 = tb * kSpmvTile - i0;
  const int rp_first = i0 < N ? __ldg(row_ptr + i0) : E;
  bool head_pending = i0 < N && rp_first < j0;  // row i0 began in an earlier warp's range
  float carry = 0.f;

  // row ends (row_ptr[i+1]) and column indices of a tile starting at (i, j)
  int re[kSpmvItems], ci[kSpmvItems];
  auto load_tile = [&](int i, int j) {
    const int* rp = row_ptr + i + 1 + lane;
    const int* cp = col + j + lane;
    if (i + kSpmvTile <= N && j + kSpmvTile <= E) {  // interior tile: no bounds checks
#pragma unroll
      for (int u = 0; u < kSpmvItems; ++u) {
        re[u] = spmv_ld_stream<XP, SP>(rp + 32 * u, pol_stream);
        ci[u] = spmv_ld_stream<XP, SP>(cp + 32 * u, pol_stream);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kSpmvItems; ++u) {
        const int p = lane + 32 * u;
        re[u] = i + p < N ? spmv_ld_stream<XP, SP>(rp + 32 * u, pol_stream) : 0x3fffffff;
        ci[u] = j + p < E ? spmv_ld_stream<XP, SP>(cp + 32 * u, pol_stream) : 0;
      }
    }
  };
  load_tile(i0, j0);

  for (int c = tb; c < te; ++c) {
    const int L = min(total - c * kSpmvTile, kSpmvTile);
    // ---- 1. rows ending in this tile: pos(p) = p + row_ptr[i0+p+1] - j0 < L
    int pos[kSpmvItems];
    int nr = 0;
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u) {
      pos[u] = lane + 32 * u + (re[u] - j0);
      nr += __popc(__ballot_sync(0xffffffffu, pos[u] < L));
    }
    const int i1 = i0 + nr, j1 = j0 + (L - nr);
    const int nn = L - nr;
    // ---- 2. gathers; then the next tile's row ends and columns go in flight
    float xv[kSpmvItems];
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u)
      xv[u] = lane + 32 * u < nn ? spmv_ld_x<XP>(x + ci[u], pol_keep) : 0.f;
    if (c + 1 < te) load_tile(i1, j1);
    // ---- 3. row-end marks and gathered values to shared memory
    __syncwarp();  // the previous tile's shared-memory reads are done
    reinterpret_cast<uint2*>(s_mark)[lane] = make_uint2(0u, 0u);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u)
      if (pos[u] < L) s_mark[pos[u]] = 1;
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u) s_val[lane + 32 * u] = xv[u];  // zeros past nn
    __syncwarp();
    // 8 mark bytes (0/1) -> 8 flag bits: (w * 0x01020408) >> 24 packs a word's 4 bytes
    const uint2 mw = reinterpret_cast<const uint2*>(s_mark)[lane];
    const unsigned fl = ((mw.x * 0x01020408u) >> 24) | (((mw.y * 0x01020408u) >> 24) << 4);
    const int cnt = __popc(fl);
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    int ri = incl - cnt;                       // local index of this lane's first row end
    const int nj0 = lane * kSpmvItems - ri;    // local index of its first non-zero
    // items past the tile's end carry no mark and read zeros (s_val past nn)
    float v[kSpmvItems];
#pragma unroll
    for (int k = 0; k < kSpmvItems; ++k) v[k] = s_val[nj0 + k - __popc(fl & ((1u << k) - 1u))];
    float sum = 0.f, first_val = 0.f;
    int first_row = -1;
#pragma unroll
    for (int k = 0; k < kSpmvItems; ++k) {
      if ((fl >> k) & 1u) {
        if (first_row < 0) { first_row = ri; first_val = sum; }
        else s_y[ri] = sum;
        sum = 0.f;
        ++ri;
      } else {
        sum += v[k];
      }
    }
    // ---- 4. segmented scan across lanes, carry across tiles
    float sc = sum;
    bool f = first_row >= 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float yv = __shfl_up_sync(0xffffffffu, sc, off);
      const bool fv = __shfl_up_sync(0xffffffffu, f, off);
      if (lane >= off && !f) { sc += yv; f = fv; }
    }
    const float acc = f ? sc : sc + carry;  // running value of the open row at this lane
    const float prev = __shfl_up_sync(0xffffffffu, acc, 1);
    if (first_row >= 0) s_y[first_row] = first_val + (lane == 0 ? carry : prev);
    carry = __shfl_sync(0xffffffffu, acc, 31);
    __syncwarp();
    int pstart = 0;
    if (head_pending && nr > 0) {
      spmv_deposit(ws, y, i0, warp_of_diag((long long)i0 + rp_first), g, g, s_y[0], true);
      head_pending = false;
      pstart = 1;
    }
    float* yo = y + i0;
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u) {
      const int p = lane + 32 * u;
      if (p >= pstart && p < nr) {
        if (SP == 0) yo[p] = s_y[p];
        else stg_hint(yo + p, s_y[p], pol_stream);
      }
    }
    i0 = i1;
    j0 = j1;
  }
  // the row crossing this range's end: deposit this warp's share
  if (i0 < N) {
    const long long rs = __ldg(row_ptr + i0), rend = __ldg(row_ptr + i0 + 1);
    const long long as = warp_of_diag(i0 + rs), ae = warp_of_diag(i0 + rend);
    if (ae > g && as <= g) spmv_deposit(ws, y, i0, as, ae, g, carry, false);
  }
}

// Version with the gathers one tile ahead: x[col] values of tile c+1 are
// copied by 4-byte cp.async straight into the warp's second s_val buffer
// while tile c is reduced, so the gather latency leaves the per-tile
// critical path without costing registers.  Same arithmetic (bit-identical
// results) as spmv_body.
template <int SP>
__device__ __forceinline__ void spmv_body_async(const int* __restrict__ row_ptr,
                                                const int* __restrict__ col,
                                                const float* __restrict__ x, float* __restrict__ y,
                                                long long N_) {
  __shared__ float s_val_all[kSpmvWarps][2][kSpmvTile];
  __shared__ float s_y_all[kSpmvWarps][kSpmvTile];
  __shared__ __align__(16) unsigned char s_mark_all[kSpmvWarps][kSpmvTile];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* s_y = s_y_all[warp];
  unsigned char* s_mark = s_mark_all[warp];
  const long long E_ = (long long)__ldg(row_ptr + N_);
  if (N_ + E_ + kSpmvTile >= (1ll << 31)) __trap();  // merge coordinates are 32-bit (documented limit)
  const int N = (int)N_, E = (int)E_, total = N + E;
  const int ntiles = (total + kSpmvTile - 1) / kSpmvTile;
  const int G = (int)gridDim.x * kSpmvWarps;
  const int g = (int)blockIdx.x * kSpmvWarps + warp;
  const int per = (ntiles + G - 1) / G;
  const int tb = g * per, te = min(ntiles, tb + per);
  if (tb >= te) return;  // warp-uniform; the kernel has no CTA barriers
  const SpmvWs ws = spmv_ws(y, N_, G);
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  auto warp_of_diag = [&](long long d) { return (d / kSpmvTile) / per; };

  int i0 = (int)warp_merge_search(row_ptr, N_, E_, (long long)tb * kSpmvTile);
  int j0 = tb * kSpmvTile - i0;
  const int rp_first = i0 < N ? __ldg(row_ptr + i0) : E;
  bool head_pending = i0 < N && rp_first < j0;  // row i0 began in an earlier warp's range
  float carry = 0.f;

  int re[kSpmvItems], ci[kSpmvItems];
  auto load_tile = [&](int i, int j) {
    const int* rp = row_ptr + i + 1 + lane;
    const int* cp = col + j + lane;
    if (i + kSpmvTile <= N && j + kSpmvTile <= E) {
#pragma unroll
      for (int u = 0; u < kSpmvItems; ++u) {
        re[u] = spmv_ld_stream<1, SP>(rp + 32 * u, pol_stream);
        ci[u] = spmv_ld_stream<1, SP>(cp + 32 * u, pol_stream);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kSpmvItems; ++u) {
        const int p = lane + 32 * u;
        re[u] = i + p < N ? spmv_ld_stream<1, SP>(rp + 32 * u, pol_stream) : 0x3fffffff;
        ci[u] = j + p < E ? spmv_ld_stream<1, SP>(cp + 32 * u, pol_stream) : 0;
      }
    }
  };
  // merge positions of the row ends in a tile starting at (i, j) with re[] loaded;
  // returns the number of rows ending in it
  auto row_ends = [&](int j, int L, int (&pos)[kSpmvItems]) {
    int nr = 0;
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u) {
      pos[u] = lane + 32 * u + (re[u] - j);
      nr += __popc(__ballot_sync(0xffffffffu, pos[u] < L));
    }
    return nr;
  };
  // gathers of a tile with nn non-zeros into buffer b (zero-filled past nn), one commit group
  auto gather = [&](int nn, int b) {
    float* dst = s_val_all[warp][b];
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u) {
      const int k = lane + 32 * u;
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + k);
      const float* src = k < nn ? x + ci[u] : x;
      asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2, %3;" ::"r"(d),
                   "l"(src), "r"(k < nn ? 4 : 0), "l"(pol_keep)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // prologue: tile tb's row ends and gathers, tile tb+1's indices in flight
  load_tile(i0, j0);
  int pos[kSpmvItems];
  int L = min(total - tb * kSpmvTile, kSpmvTile);
  int nr = row_ends(j0, L, pos);
  int i1 = i0 + nr, j1 = j0 + (L - nr);
  gather(L - nr, 0);
  if (tb + 1 < te) load_tile(i1, j1);

  for (int c = tb; c < te; ++c) {
    const int b = (c - tb) & 1;
    // ---- next tile: row ends, gathers (cp.async, other buffer), indices of the one after
    int posn[kSpmvItems];
    int Ln = 0, nrn = 0;
    __syncwarp();  // all lanes finished reading buffer b^1 (tile c-1)
    if (c + 1 < te) {
      Ln = min(total - (c + 1) * kSpmvTile, kSpmvTile);
      nrn = row_ends(j1, Ln, posn);
      gather(Ln - nrn, b ^ 1);
      if (c + 2 < te) load_tile(i1 + nrn, j1 + (Ln - nrn));
    } else {
      asm volatile("cp.async.commit_group;" ::: "memory");  // keep one group per step
    }
    // ---- tile c: marks, then wait for its gathers
    reinterpret_cast<uint2*>(s_mark)[lane] = make_uint2(0u, 0u);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u)
      if (pos[u] < L) s_mark[pos[u]] = 1;
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const float* s_val = s_val_all[warp][b];
    const uint2 mw = reinterpret_cast<const uint2*>(s_mark)[lane];
    const unsigned fl = ((mw.x * 0x01020408u) >> 24) | (((mw.y * 0x01020408u) >> 24) << 4);
    const int cnt = __popc(fl);
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    int ri = incl - cnt;
    const int nj0 = lane * kSpmvItems - ri;
    float v[kSpmvItems];
#pragma unroll
    for (int k = 0; k < kSpmvItems; ++k) v[k] = s_val[nj0 + k - __popc(fl & ((1u << k) - 1u))];
    float sum = 0.f, first_val = 0.f;
    int first_row = -1;
#pragma unroll
    for (int k = 0; k < kSpmvItems; ++k) {
      if ((fl >> k) & 1u) {
        if (first_row < 0) { first_row = ri; first_val = sum; }
        else s_y[ri] = sum;
        sum = 0.f;
        ++ri;
      } else {
        sum += v[k];
      }
    }
    float sc = sum;
    bool f = first_row >= 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float yv = __shfl_up_sync(0xffffffffu, sc, off);
      const bool fv = __shfl_up_sync(0xffffffffu, f, off);
      if (lane >= off && !f) { sc += yv; f = fv; }
    }
    const float acc = f ? sc : sc + carry;
    const float prev = __shfl_up_sync(0xffffffffu, acc, 1);
    if (first_row >= 0) s_y[first_row] = first_val + (lane == 0 ? carry : prev);
    carry = __shfl_sync(0xffffffffu, acc, 31);
    __syncwarp();
    int pstart = 0;
    if (head_pending && nr > 0) {
      spmv_deposit(ws, y, i0, warp_of_diag((long long)i0 + rp_first), g, g, s_y[0], true);
      head_pending = false;
      pstart = 1;
    }
    float* yo = y + i0;
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u) {
      const int p = lane + 32 * u;
      if (p >= pstart && p < nr) {
        if (SP == 0) yo[p] = s_y[p];
        else stg_hint(yo + p, s_y[p], pol_stream);
      }
    }
    // advance: tile c+1 becomes current
    i0 = i1;
    j0 = j1;
    i1 = i0 + nrn;
    j1 = j0 + (Ln - nrn);
    L = Ln;
    nr = nrn;
#pragma unroll
    for (int u = 0; u < kSpmvItems; ++u) pos[u] = posn[u];
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (i0 < N) {
    const long long rs = __ldg(row_ptr + i0), rend = __ldg(row_ptr + i0 + 1);
    const long long as = warp_of_diag(i0 + rs), ae = warp_of_diag(i0 + rend);
    if (ae > g && as <= g) spmv_deposit(ws, y, i0, as, ae, g, carry, false);
  }
}

#define SPMV_VARIANT(NAME, XP, SP)                                                                 \
  __global__ void __launch_bounds__(kSpmvThreads, 4)                                               \
      NAME(const int* __restrict__ row_ptr, const int* __restrict__ col, const float* __restrict__ x, \
           float* __restrict__ y, long long N) {                                                     \
    spmv_body<XP, SP>(row_ptr, col, x, y, N);                                                        \
  }
SPMV_VARIANT(k_spmv_sync, 1, 2)
SPMV_VARIANT(k_spmv_x0s1, 0, 1)
SPMV_VARIANT(k_spmv_x1s1, 1, 1)
#define SPMV_ASYNC_VARIANT(NAME, SP)                                                               \
  __global__ void __launch_bounds__(kSpmvThreads, 4)                                               \
      NAME(const int* __restrict__ row_ptr, const int* __restrict__ col, const float* __restrict__ x, \
           float* __restrict__ y, long long N) {                                                     \
    spmv_body_async<SP>(row_ptr, col, x, y, N);                                                      \
  }
SPMV_ASYNC_VARIANT(k_spmv, 2)
SPMV_ASYNC_VARIANT(k_spmv_as1, 1)


// ---------------------------------------------------------------------------
// SpMV by row class ("spmv_plan"; an alternative to the merge-path kernel,
// which stays the product kernel: on the HITS graph this one measured 375 us
// in its first, one-CTA-per-unit form (thresholds 8/4096/8192) and 420-490 us
// in the form below, vs 362 us for merge-path -- tools/spmv_footprint.py).
//
// On the 20M-vertex power-law graph the merge-path kernels above run at
// ~300 us whatever the gather footprint (tools/spmv_footprint.py: folding
// the columns into N/64 entries saves only 18%).  The idea here: split the
// rows by degree once, when the graph is
// registered (a small "plan" array built from row_ptr, spmv_plan() in
// programs/hits_dl.py), and each class gets the cheapest exact schedule:
//   * short rows (deg <= 4; ~95% of rows): one thread per row, 4 rows per
//     thread 256 apart (coalesced row_ptr reads and y writes), the column
//     loads of all 4 rows then all their gathers in flight, each row summed
//     in column order;
//   * medium rows (4 < deg <= 256): 8 lanes per row, 4 rows per warp, 8
//     column loads then 8 gathers in flight per lane, fixed xor-tree sum;
//   * long rows (deg > 256; ~10^4 hubs holding ~half of the non-zeros):
//     chunks of 2048 non-zeros, one CTA per chunk (8 loads in flight per
//     thread, block reduction in a fixed tree); a hub's chunk sums are added
//     in chunk order by the last chunk to arrive (atomic arrival count), so
//     results are bit-reproducible.
// One launch = one DAG vertex; a persistent grid walks the units (long
// chunks first, then medium-row groups, then short-row blocks).
// Workspace after y's N floats (16-byte aligned): NL chunk sums, NL
// arrival counters (zero at allocation; reset by the last arriver).
constexpr int kPlanHeader = 16;    // [0] NL long chunks, [1] NM medium rows, [2] NS short blocks
constexpr int kShortMax = 4;       // deg <= 4: thread per row
constexpr int kLongMin = 256;      // deg > 256: CTA per chunk of kLongChunk non-zeros
constexpr int kLongChunk = 2048;
constexpr int kShortRowsPerThread = 4;
constexpr int kShortRowsPerCta = 256 * kShortRowsPerThread;
constexpr int kMedRowsPerCta = 32;  // 8 warps x 4 groups of 8 lanes

// HINT 1: L2 evict-first for the streamed column indices, evict-last for the gathers
template <int HINT>
__device__ __forceinline__ float spmv_gather(const float* x, int c, uint64_t pol) {
  return HINT ? ldg_hint(x + c, pol) : __ldg(x + c);
}
template <int HINT>
__device__ __forceinline__ int spmv_col(const int* col, int k, uint64_t pol) {
  return HINT ? ldg_hint(col + k, pol) : __ldg(col + k);
}

// Persistent: CTA b takes units b, b + G, b + 2G, ... of the unit list
// [NL long chunks | ceil(NM/32) medium groups | NS short blocks].  Every
// path issues all of a unit's index loads, then all its gathers, before
// using any (memory-level parallelism: the chains row_ptr -> col -> x are
// the cost, not the arithmetic).
template <int HINT>
__device__ __forceinline__ void spmv_plan_body(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                               const int* __restrict__ plan, const float* __restrict__ x,
                                               float* __restrict__ y, long long N_) {
  __shared__ float sh[32];
  __shared__ bool last;
  uint64_t pcol = 0, px = 0;
  if (HINT) {
    pcol = l2_policy_evict_first();
    px = l2_policy_evict_last();
  }
  const int NL = __ldg(plan + 0), NM = __ldg(plan + 1), NS = __ldg(plan + 2);
  // the plan must have been built with this kernel's class bounds
  if (__ldg(plan + 3) != kShortMax || __ldg(plan + 4) != kLongMin || __ldg(plan + 5) != kLongChunk) __trap();
  const int NMC = (NM + kMedRowsPerCta - 1) / kMedRowsPerCta;
  const int units = NL + NMC + NS;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int N = (int)N_;
  uintptr_t wsb = ((uintptr_t)(y + N) + 15) & ~(uintptr_t)15;
  float* part = reinterpret_cast<float*>(wsb);
  unsigned* arrive = reinterpret_cast<unsigned*>(part + NL);
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    if (u < NL) {
      // ---- long-row chunk: (row, k_begin, first chunk of the row, chunks of the row)
      const int4 it = __ldg(reinterpret_cast<const int4*>(plan + kPlanHeader) + u);
      const int row = it.x, kb = it.y, first = it.z, cnt = it.w;
      const int ke = min(kb + kLongChunk, __ldg(row_ptr + row + 1));
      // unconditional loads at clamped (valid) addresses, results selected:
      // keeps all 8 column loads, then all 8 gathers, in flight
      int c[kLongChunk / 256];
#pragma unroll
      for (int q = 0; q < kLongChunk / 256; ++q) {
        const int k = kb + t + q * 256;
        c[q] = spmv_col<HINT>(col, k < ke ? k : kb, pcol);
      }
      float v[kLongChunk / 256];
#pragma unroll
      for (int q = 0; q < kLongChunk / 256; ++q) v[q] = spmv_gather<HINT>(x, c[q], px);
      float a = 0.f;
#pragma unroll
      for (int q = 0; q < kLongChunk / 256; ++q) a += kb + t + q * 256 < ke ? v[q] : 0.f;
      const float sum = block_reduce(a, OpAdd(), sh);
      if (cnt == 1) {
        if (t == 0) y[row] = sum;
        continue;
      }
      if (t == 0) {
        part[u] = sum;
        __threadfence();
        last = atomicAdd(arrive + first, 1u) == (unsigned)(cnt - 1);
      }
      __syncthreads();
      if (last && warp == 0) {  // chunk sums of the row in chunk order
        __threadfence();
        const volatile float* vp = part;
        float w = 0.f;
        for (int i = lane; i < cnt; i += 32) w += vp[first + i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (lane == 0) {
          y[row] = w;
          arrive[first] = 0;  // reusable by the next launch
        }
      }
      __syncthreads();  // `last` is rewritten by the next chunk unit
      continue;
    }
    if (u < NL + NMC) {
      // ---- medium rows: 8 lanes per row, 4 rows per warp
      const int m = (u - NL) * kMedRowsPerCta + warp * 4 + (lane >> 3);
      const int sub = lane & 7;
      int kb = 0, ke = 0, row = -1;
      if (m < NM) {
        row = __ldg(plan + kPlanHeader + 4 * NL + m);
        kb = __ldg(row_ptr + row);
        ke = __ldg(row_ptr + row + 1);
      }
      float acc = 0.f;
      for (int k0 = kb + sub; k0 < ke; k0 += 8 * 8) {
        int c[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) c[q] = spmv_col<HINT>(col, k0 + q * 8 < ke ? k0 + q * 8 : kb, pcol);
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = spmv_gather<HINT>(x, c[q], px);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += k0 + q * 8 < ke ? v[q] : 0.f;
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (sub == 0 && row >= 0) y[row] = acc;
      continue;
    }
    // ---- short rows: thread per row, 4 rows per thread 256 apart; all column
    // loads of the 4 rows, then all their gathers
    const int r0 = (u - NL - NMC) * kShortRowsPerCta + t;
    int b[kShortRowsPerThread], d[kShortRowsPerThread];
#pragma unroll
    for (int j = 0; j < kShortRowsPerThread; ++j) {
      const int r = r0 + 256 * j;
      b[j] = r < N ? __ldg(row_ptr + r) : 0;
      d[j] = r < N ? __ldg(row_ptr + r + 1) - b[j] : 0;
      if (d[j] > kShortMax) d[j] = -1;  // medium / long row: summed by its own unit
    }
    // the first two non-zeros of every row: unconditional loads at valid
    // addresses (col[0], x[0] when absent), 8 + 8 in flight per thread; the
    // rarer third and fourth under a branch
    int c[kShortRowsPerThread][kShortMax];
#pragma unroll
    for (int j = 0; j < kShortRowsPerThread; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) c[j][q] = spmv_col<HINT>(col, q < d[j] ? b[j] + q : 0, pcol);
#pragma unroll
    for (int j = 0; j < kShortRowsPerThread; ++j)
#pragma unroll
      for (int q = 2; q < kShortMax; ++q) c[j][q] = q < d[j] ? spmv_col<HINT>(col, b[j] + q, pcol) : 0;
    float v[kShortRowsPerThread][kShortMax];
#pragma unroll
    for (int j = 0; j < kShortRowsPerThread; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) v[j][q] = spmv_gather<HINT>(x, q < d[j] ? c[j][q] : 0, px);
#pragma unroll
    for (int j = 0; j < kShortRowsPerThread; ++j)
#pragma unroll
      for (int q = 2; q < kShortMax; ++q) v[j][q] = q < d[j] ? spmv_gather<HINT>(x, c[j][q], px) : 0.f;
#pragma unroll
    for (int j = 0; j < kShortRowsPerThread; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) v[j][q] = q < d[j] ? v[j][q] : 0.f;
#pragma unroll
    for (int j = 0; j < kShortRowsPerThread; ++j) {
      const int r = r0 + 256 * j;
      float sum = 0.f;
#pragma unroll
      for (int q = 0; q < kShortMax; ++q) sum += v[j][q];
      if (r < N && d[j] >= 0) y[r] = sum;
    }
  }
}

__global__ void __launch_bounds__(256) k_spmv_plan(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                   const int* __restrict__ plan, const float* __restrict__ x,
                                                   float* __restrict__ y, long long N) {
  spmv_plan_body<0>(row_ptr, col, plan, x, y, N);
}
__global__ void __launch_bounds__(256) k_spmv_plan_h(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                     const int* __restrict__ plan, const float* __restrict__ x,
                                                     float* __restrict__ y, long long N) {
  spmv_plan_body<1>(row_ptr, col, plan, x, y, N);
}

// ---------------------------------------------------------------------------
// NON-ZERO-SPLIT SpMV ("spmv_nz", the product kernel since round 2).
//
// Measured bound on the HITS graph (tools/spmv_lab.py, profiles/r2_spmv_lab*):
// the 54M random 4-byte gathers alone, with the column stream, take 177 us
// (~1.1 gathers per SM per clock: one L1 wavefront per divergent lane), the
// column stream alone 35 us; the merge-path kernel above took 364 us, i.e.
// half its time went to the row structure (merge search, marks, row-end
// scans over N + E items, 45% of the rows being empty).  This kernel walks
// the NON-ZEROS only, in chunks of 128 (4 per lane, one 128-bit column load
// per lane, 4 gathers in flight), with the row structure re-encoded once when
// the graph is registered (spmv_nz_plan() in programs/hits_dl.py; the graph
// is static and resident):
//   flags[]  1 bit per non-zero: it starts a (non-empty) row;
//   nzrow[]  the ids of the non-empty rows, in order (ordinals -> row ids);
//   rbase[]  ordinal of the row holding each chunk's first non-zero.
// Per chunk a lane sums its items per row segment, a segmented warp scan
// carries open rows across lanes (and a register across the warp's chunks),
// and every completed row is written by the lane where it ends, together
// with the zeros of the empty rows just before it.  Global warp g owns the
// contiguous chunk range [g*per, (g+1)*per): equal non-zeros per warp
// whatever the degree distribution.  A row spanning several warp ranges is
// finished by the last of its participants to deposit its share (atomic
// arrival count; shares added in warp order) -> bit-reproducible, no float
// atomics.  Column indices are streamed with L1::no_allocate and L2
// evict_first so that L1 and L2 keep the gathered vector (lab: 177 vs 184 us
// for plain loads).  row_ptr is read only for rows crossing warp ranges.
// Workspace after y's N floats: SpmvWs (3 words per warp of the grid).
constexpr int kNzMagic = 0x4e5a3031;  // "NZ01"

struct NzPlan {
  int nc, nr;           // chunks, non-empty rows
  const int* rbase;     // [nc + 1]
  const unsigned* flags;  // [ceil(E / 32) + 4]
  const int* nzrow;     // [nr]
};

__device__ __forceinline__ NzPlan nz_plan(const int* plan) {
  if (__ldg(plan) != kNzMagic || __ldg(plan + 3) != kNzChunk) __trap();  // built for another kernel
  NzPlan P;
  P.nc = __ldg(plan + 1);
  P.nr = __ldg(plan + 2);
  P.rbase = plan + __ldg(plan + 4);
  P.flags = reinterpret_cast<const unsigned*>(plan + __ldg(plan + 5));
  P.nzrow = plan + __ldg(plan + 6);
  return P;
}


__device__ __forceinline__ NzIn nz_load(const int* __restrict__ col, const NzPlan& P, int chunk, int lane,
                                        int E, uint64_t pol) {
  NzIn in;
  const int k = chunk * kNzChunk + 4 * lane;
  if (k + 3 < E) {
    const int4 q = ld_cols_stream(col + k, pol);
    in.c[0] = q.x; in.c[1] = q.y; in.c[2] = q.z; in.c[3] = q.w;
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) in.c[u] = k + u < E ? __ldg(col + k + u) : -1;
  }
  in.fw = __ldg(reinterpret_cast<const uint4*>(P.flags) + chunk);  // words 4c..4c+3 (zero past E)
  return in;
}


// Software pipeline per warp: while chunk c is reduced, the column indices
// and flags of chunk c+2 and the gathers of chunk c+1 are in flight, and the
// row ids of chunk c's completed rows are loaded before its gathered values
// are consumed -- the dependent memory latencies of a chunk (indices ->
// gathers; ordinals -> row ids) overlap with the neighbouring chunks' work.
// Counting starts needs no shuffles (popc over the chunk's flag words), and
// the segmented scan shuffles only values: which lanes hold a start is one
// ballot.
__global__ void __launch_bounds__(256, 4) k_spmv_nz(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                    const int* __restrict__ plan, const float* __restrict__ x,
                                                    float* __restrict__ y, long long N_) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int N = (int)N_;
  const NzPlan P = nz_plan(plan);
  const int E = __ldg(row_ptr + N);
  const int G = (int)gridDim.x * (blockDim.x >> 5);
  const int g = (int)blockIdx.x * (blockDim.x >> 5) + warp;
  if (P.nr == 0) {  // no non-zeros: y = 0
    for (int i = g * 32 + lane; i < N; i += G * 32) y[i] = 0.f;
    return;
  }
  const int per = (P.nc + G - 1) / G;
  const int cb = g * per, ce = min(P.nc, cb + per);
  if (cb >= ce) return;  // warp-uniform; the kernel has no CTA barriers
  const SpmvWs ws = spmv_ws(y, N_, G);
  const uint64_t pol = l2_policy_evict_first();
  auto warp_of_nz = [&](int k) { return (k / kNzChunk) / per; };
  const int wsel = lane >> 3, bsh = 4 * (lane & 7);
  const unsigned lanes_below = (1u << lane) - 1u;

  // R0 = ordinal of the row open at the start of the current chunk: at the
  // range start, the row holding its first item (whose start bit, if any, is
  // consumed here); it began in an earlier warp's range unless that item
  // starts it
  const int k0w = cb * kNzChunk;
  const bool start0 = (__ldg(P.flags + (k0w >> 5)) >> (k0w & 31)) & 1u;
  int R0 = __ldg(P.rbase + cb);
  bool head_pending = !start0;
  float carry = 0.f;

  NzIn cur = nz_load(col, P, cb, lane, E, pol);
  NzIn nxt = cur;
  if (cb + 1 < ce) nxt = nz_load(col, P, cb + 1, lane, E, pol);
  float v[4];
  nz_gather(cur, x, v);
  for (int c = cb; c < ce; ++c) {
    uint4 fw = cur.fw;
    if (c == cb) fw.x &= ~1u;  // the range's first item: handled by start0/head_pending
    const unsigned mine = wsel == 0 ? fw.x : (wsel == 1 ? fw.y : (wsel == 2 ? fw.z : fw.w));
    const unsigned fl = (mine >> bsh) & 0xFu;
    // ---- ordinals of the rows completed in this lane (no dependence on the gathers)
    const int nst = __popc(fl);
    const int before = (wsel > 0 ? __popc(fw.x) : 0) + (wsel > 1 ? __popc(fw.y) : 0) +
                       (wsel > 2 ? __popc(fw.z) : 0) + __popc(mine & ((1u << bsh) - 1u));
    const int total = __popc(fw.x) + __popc(fw.y) + __popc(fw.z) + __popc(fw.w);
    const int o = R0 + before;  // the row open entering the lane; ends at its first start
    // row ids of ordinals o-1 .. o+3 (those this lane writes), in registers
    int rid0 = -1, rid1 = -1, rid2 = -1, rid3 = -1, rid4 = -1;
    if (nst) {
      rid0 = o > 0 ? __ldg(P.nzrow + o - 1) : -1;
      rid1 = __ldg(P.nzrow + o);
      if (nst > 1) rid2 = __ldg(P.nzrow + o + 1);
      if (nst > 2) rid3 = __ldg(P.nzrow + o + 2);
      if (nst > 3) rid4 = __ldg(P.nzrow + o + 3);
    }
    auto rid = [&](int j) { return j <= 1 ? (j == 0 ? rid0 : rid1) : (j == 2 ? rid2 : (j == 3 ? rid3 : rid4)); };
    // ---- next chunk's gathers and the chunk after's indices go in flight
    float vn[4] = {0.f, 0.f, 0.f, 0.f};
    if (c + 1 < ce) {
      nz_gather(nxt, x, vn);
      cur = nxt;
      if (c + 2 < ce) nxt = nz_load(col, P, c + 2, lane, E, pol);
    }
    // ---- lane-local row segments of this chunk
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
    // ---- segmented inclusive scan of the open-row contributions; the
    // segment test comes from the ballot of start-holding lanes
    const unsigned m = __ballot_sync(0xffffffffu, nst != 0);
    float sv = nst ? run : head;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float tv = __shfl_up_sync(0xffffffffu, sv, off);
      // lanes (lane-off, lane] hold no start: the open row reaches back
      const unsigned win = lane >= off ? (m >> (lane - off + 1)) & ((1u << off) - 1u) : 1u;
      if (win == 0u) sv += tv;
    }
    float cin = __shfl_up_sync(0xffffffffu, sv, 1);
    if (lane == 0) cin = 0.f;
    if ((m & lanes_below) == 0u) cin += carry;  // no start below this lane: the chunk's carry
    // ---- rows completed in this lane: y[row] = sum, zeros for the empty rows before it
    if (nst) {
      const float val = cin + head;
      if (head_pending && before == 0) {
        // began before this warp's range: deposit (this warp holds its end)
        const int cs = warp_of_nz(__ldg(row_ptr + rid1));
        spmv_ws_put(ws, g, val, true);
        if (spmv_ws_arrive(ws, cs, g)) {
          for (int r = rid0 + 1; r < rid1; ++r) y[r] = 0.f;
          y[rid1] = spmv_ws_sum(ws, cs, g);
        }
      } else {
        for (int r = rid0 + 1; r < rid1; ++r) y[r] = 0.f;
        y[rid1] = val;
      }
      int j = 1;
      float r2 = 0.f;
      bool in = false;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if ((fl >> u) & 1u) {
          if (in) {
            const int a = rid(j), b = rid(j + 1);
            for (int r = a + 1; r < b; ++r) y[r] = 0.f;
            y[b] = r2;
            ++j;
          }
          in = true;
          r2 = 0.f;
        }
        r2 += v[u];
      }
    }
    // ---- carry to the next chunk
    const float tail_all = __shfl_sync(0xffffffffu, sv, 31);
    carry = m ? tail_all : carry + tail_all;
    if (m) head_pending = false;
    R0 += total;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = vn[u];
  }
  // ---- the row open at the range end (and, for the last non-empty row, the
  // empty rows after it: no start follows the last row, so it is always
  // completed here)
  if (lane == 0) {
    const int ke = ce * kNzChunk;
    const bool ends_here = ke >= E || ((__ldg(P.flags + (ke >> 5)) >> (ke & 31)) & 1u);
    const int row = __ldg(P.nzrow + R0);
    const int prev = R0 > 0 ? __ldg(P.nzrow + R0 - 1) : -1;
    float out = carry;
    bool write = true;
    if (ends_here) {
      if (head_pending) {  // spans the whole range, ends at its end
        const int cs = warp_of_nz(__ldg(row_ptr + row));
        spmv_ws_put(ws, g, carry, true);
        write = spmv_ws_arrive(ws, cs, g);
        if (write) out = spmv_ws_sum(ws, cs, g);
      }
    } else {
      const int cs = warp_of_nz(__ldg(row_ptr + row));
      const int cend = warp_of_nz(__ldg(row_ptr + row + 1) - 1);
      spmv_ws_put(ws, g, carry, false);
      write = spmv_ws_arrive(ws, cs, cend);
      if (write) out = spmv_ws_sum(ws, cs, cend);
    }
    if (write) {
      for (int r = prev + 1; r < row; ++r) y[r] = 0.f;
      y[row] = out;
      if (R0 == P.nr - 1)
        for (int r = row + 1; r < N; ++r) y[r] = 0.f;
    }
  }
}

__global__ void __launch_bounds__(256, 4) k_spmv_pad2(const int* __restrict__, const int* __restrict__,
                                                      const int* __restrict__ plan, const float* __restrict__ x,
                                                      float* __restrict__ y, long long N_) {
  spmv_pad2_body<4>(plan, x, y, N_);
}
__global__ void __launch_bounds__(256, 3) k_spmv_pad2b3(const int* __restrict__, const int* __restrict__,
                                                        const int* __restrict__ plan, const float* __restrict__ x,
                                                        float* __restrict__ y, long long N_) {
  spmv_pad2_body<3>(plan, x, y, N_);
}

// spmv_hub*: the product body with the hub head of x staged in shared memory
// (spmv_common.cuh HUB); H = dynamic shared memory / 4 per launch; 256 x 4,
// 512 x 2 and 1024 x 1 threads per SM (the same 64-register budget).
__global__ void __launch_bounds__(256, 4) k_spmv_hub4(const int* __restrict__, const int* __restrict__,
                                                      const int* __restrict__ plan, const float* __restrict__ x,
                                                      float* __restrict__ y, long long N_) {
  spmv_pad2_body<4, true>(plan, x, y, N_);
}
__global__ void __launch_bounds__(512, 2) k_spmv_hub2(const int* __restrict__, const int* __restrict__,
                                                      const int* __restrict__ plan, const float* __restrict__ x,
                                                      float* __restrict__ y, long long N_) {
  spmv_pad2_body<2, true>(plan, x, y, N_);
}
__global__ void __launch_bounds__(1024, 1) k_spmv_hub1(const int* __restrict__, const int* __restrict__,
                                                       const int* __restrict__ plan, const float* __restrict__ x,
                                                       float* __restrict__ y, long long N_) {
  spmv_pad2_body<1, true>(plan, x, y, N_);
}

// ---------------------------------------------------------------------------
// spmv_ws: the padded non-zero split with the gathers and the row logic on
// DIFFERENT warps.  ncu on the product (profiles/r2_*): the gathers are
// bounded by the L1/L2 request rate (lab floor 177 us for the 57M gathers +
// the column stream), and each warp's chunk carries a long dependent chain
// (flags -> popc -> ballot -> 5-step shuffle scan -> stores) that leaves the
// request pipe idle when all warps of a scheduler sit in their chains.  Here
// a CTA holds 4 producer warps that only load columns and gather x into a
// per-pair shared ring (TWO chunks per step: 8 gathers in flight per lane),
// and 4 consumer warps that reduce the staged values exactly like the
// product (same rows, same deposits, same summation order: bit-identical).
// Producer p serves consumer p over the consumer's chunk range; each ring
// slot has a full and an empty mbarrier (32 arrivals each: every lane
// arrives after its own shared-memory accesses).
constexpr int kWsPairs = 4;     // producer/consumer warp pairs per CTA
constexpr int kWsSlots = 8;     // ring slots per pair (one chunk each)
struct WsSlot {
  float4 v[32];   // the chunk's 128 gathered values, lane-major
  uint4 fw;       // its 4 flag words
};
__device__ __forceinline__ void ws_mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void ws_mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}
__device__ __forceinline__ void ws_mbar_wait(uint64_t* b, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(256, 4) k_spmv_ws(const int* __restrict__, const int* __restrict__,
                                                    const int* __restrict__ plan, const float* __restrict__ x,
                                                    float* __restrict__ y, long long N_) {
  __shared__ WsSlot ring[kWsPairs][kWsSlots];
  __shared__ uint64_t full[kWsPairs][kWsSlots], empty[kWsPairs][kWsSlots];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pair = warp & (kWsPairs - 1);
  const bool producer = warp >= kWsPairs;
  if (threadIdx.x < kWsPairs * kWsSlots) {
    ws_mbar_init(&full[0][0] + threadIdx.x, 32);
    ws_mbar_init(&empty[0][0] + threadIdx.x, 32);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const PadPlan P = pad_plan(plan);
  if ((long long)P.n != N_ || P.n == 0 || blockDim.x != 2 * 32 * kWsPairs) return;
  const int G = (int)gridDim.x * kWsPairs;  // consumer warps of the grid
  const int g = (int)blockIdx.x * kWsPairs + pair;
  const int per = (P.nc + G - 1) / G;
  const int cb = g * per, ce = min(P.nc, cb + per);
  if (cb >= ce) return;  // both warps of the pair leave together; no CTA barrier below
  WsSlot* R = ring[pair];
  if (producer) {
    const uint64_t pol = l2_policy_evict_first();
    int it = 0;
    for (int c = cb; c < ce; c += 2, it += 2) {
      const bool two = c + 1 < ce;
      NzIn a = pad_load(P, c, lane, pol), b = a;
      if (two) b = pad_load(P, c + 1, lane, pol);
      float va[4], vb[4];
      nz_gather(a, x, va);
      if (two) nz_gather(b, x, vb);
      const int s0 = it % kWsSlots, s1 = (it + 1) % kWsSlots;
      if (it >= kWsSlots) ws_mbar_wait(&empty[pair][s0], (unsigned)((it / kWsSlots - 1) & 1));
      R[s0].v[lane] = make_float4(va[0], va[1], va[2], va[3]);
      if (lane == 0) R[s0].fw = a.fw;
      ws_mbar_arrive(&full[pair][s0]);
      if (two) {
        if (it + 1 >= kWsSlots) ws_mbar_wait(&empty[pair][s1], (unsigned)(((it + 1) / kWsSlots - 1) & 1));
        R[s1].v[lane] = make_float4(vb[0], vb[1], vb[2], vb[3]);
        if (lane == 0) R[s1].fw = b.fw;
        ws_mbar_arrive(&full[pair][s1]);
      }
    }
    return;
  }
  // consumer: the product's per-chunk reduction on staged values
  const SpmvWs ws = spmv_ws(y, N_, G);
  auto warp_of_item = [&](int k) { return (k / kNzChunk) / per; };
  const int wsel = lane >> 3, bsh = 4 * (lane & 7);
  const unsigned lanes_below = (1u << lane) - 1u;
  const int k0w = cb * kNzChunk;
  const bool start0 = (__ldg(P.flags + (k0w >> 5)) >> (k0w & 31)) & 1u;
  int R0 = __ldg(P.rbase + cb);
  bool head_pending = !start0;
  float carry = 0.f;
  int it = 0;
  for (int c = cb; c < ce; ++c, ++it) {
    const int sl = it % kWsSlots;
    ws_mbar_wait(&full[pair][sl], (unsigned)((it / kWsSlots) & 1));
    const float4 q = R[sl].v[lane];
    uint4 fw = R[sl].fw;
    ws_mbar_arrive(&empty[pair][sl]);
    float v[4] = {q.x, q.y, q.z, q.w};
    if (c == cb) fw.x &= ~1u;
    const unsigned mine = wsel == 0 ? fw.x : (wsel == 1 ? fw.y : (wsel == 2 ? fw.z : fw.w));
    const unsigned fl = (mine >> bsh) & 0xFu;
    const int nst = __popc(fl);
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
    const float tail_all = __shfl_sync(0xffffffffu, sv, 31);
    carry = m ? tail_all : carry + tail_all;
    if (m) head_pending = false;
    R0 += total;
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

__global__ void __launch_bounds__(256, 4) k_spmv_pad_l2(const int* __restrict__, const int* __restrict__,
                                                        const int* __restrict__ plan, const float* __restrict__ x,
                                                        float* __restrict__ y, long long N_) {
  spmv_pad_body<true>(plan, x, y, N_);
}

__global__ void __launch_bounds__(256, 4) k_spmv_pad(const int* __restrict__, const int* __restrict__,
                                                     const int* __restrict__ plan, const float* __restrict__ x,
                                                     float* __restrict__ y, long long N_) {
  spmv_pad_body<false>(plan, x, y, N_);
}

// ---------------------------------------------------------------------------
// spmv_tma: the product's scan-light padded split with the column-index and
// flag streams fed by the TMA unit.  ncu on the product: the warps stall on
// the register copy of the NEXT chunk's column indices (long_scoreboard: the
// column loads queue behind the gathers in the L1 request pipe, and with a
// 64-register budget only one chunk of columns can be in flight).  Here lane
// 0 of each warp keeps S chunks of columns + flags in flight with bulk copies
// into a per-warp shared ring (no registers, no L1 request slots); lanes
// read their 4 columns with one 16-byte shared load.  Needs whole chunks in
// the plan (spmv_pad_plan pads ci2 to a multiple of 128).
template <int S>
__device__ __forceinline__ void spmv_tma_body(const int* __restrict__ plan, const float* __restrict__ x,
                                              float* __restrict__ y, long long N_) {
  __shared__ __align__(128) int4 cring[8][S][32];   // 8 warps x S chunks x 128 columns
  __shared__ __align__(16) uint4 fring[8][S];
  __shared__ uint64_t bar[8][S];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const PadPlan P = pad_plan(plan);
  if ((long long)P.n != N_ || P.n == 0 || blockDim.x != 256) return;
  const int G = (int)gridDim.x * 8;
  const int g = (int)blockIdx.x * 8 + warp;
  const int per = (P.nc + G - 1) / G;
  const int cb = g * per, ce = min(P.nc, cb + per);
  if (cb >= ce) return;
  if (lane == 0) {
    for (int q = 0; q < S; ++q) bs_mbar_init(&bar[warp][q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int chunk, int slot) {  // lane 0
    uint64_t* b = &bar[warp][slot];
    const unsigned ba = (unsigned)__cvta_generic_to_shared(b);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(528u) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&cring[warp][slot][0])),
                 "l"(P.ci2 + (size_t)chunk * kNzChunk), "r"(ba)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&fring[warp][slot])),
                 "l"(P.flags + 4 * (size_t)chunk), "r"(ba)
                 : "memory");
  };
  if (lane == 0)
    for (int q = 0; q < S && cb + q < ce; ++q) issue(cb + q, q);
  const SpmvWs ws = spmv_ws(y, N_, G);
  auto warp_of_item = [&](int k) { return (k / kNzChunk) / per; };
  const int wsel = lane >> 3, bsh = 4 * (lane & 7);
  const unsigned lanes_below = (1u << lane) - 1u;
  const int k0w = cb * kNzChunk;
  const bool start0 = (__ldg(P.flags + (k0w >> 5)) >> (k0w & 31)) & 1u;
  int R0 = __ldg(P.rbase + cb);
  bool head_pending = !start0;
  float carry = 0.f, carry_lane = 0.f;
  bool dist = false;
  // take chunk `it` (the it-th of this warp) out of the ring: its columns
  // (4 per lane) and flag words; lane 0 refills the slot with chunk it + S
  auto take = [&](int it, int4& cols, uint4& fw) {
    const int slot = it % S;
    bs_mbar_wait(&bar[warp][slot], (unsigned)((it / S) & 1));
    cols = cring[warp][slot][lane];
    fw = fring[warp][slot];
    __syncwarp();
    if (lane == 0 && cb + it + S < ce) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(cb + it + S, slot);
    }
  };
  auto gather = [&](const int4& q, float (&v)[4]) {
    v[0] = q.x >= 0 ? __ldg(x + q.x) : 0.f;
    v[1] = q.y >= 0 ? __ldg(x + q.y) : 0.f;
    v[2] = q.z >= 0 ? __ldg(x + q.z) : 0.f;
    v[3] = q.w >= 0 ? __ldg(x + q.w) : 0.f;
  };
  int4 q;
  uint4 fwc, fwn = make_uint4(0, 0, 0, 0);
  take(0, q, fwc);
  float v[4];
  gather(q, v);
  for (int c = cb, it = 0; c < ce; ++c, ++it) {
    float vn[4] = {0.f, 0.f, 0.f, 0.f};
    if (c + 1 < ce) {
      take(it + 1, q, fwn);
      gather(q, vn);
    }
    uint4 fw = fwc;
    if (c == cb) fw.x &= ~1u;
    const unsigned mine = wsel == 0 ? fw.x : (wsel == 1 ? fw.y : (wsel == 2 ? fw.z : fw.w));
    const unsigned fl = (mine >> bsh) & 0xFu;
    const int nst = __popc(fl);
    const unsigned m = __ballot_sync(0xffffffffu, nst != 0);
    if (m == 0u) {
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
      if (m == 0xffffffffu) {
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
    fwc = fwn;
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
__global__ void __launch_bounds__(256, 4) k_spmv_tma4(const int* __restrict__, const int* __restrict__,
                                                      const int* __restrict__ plan, const float* __restrict__ x,
                                                      float* __restrict__ y, long long N_) {
  spmv_tma_body<4>(plan, x, y, N_);
}
__global__ void __launch_bounds__(256, 4) k_spmv_tma8(const int* __restrict__, const int* __restrict__,
                                                      const int* __restrict__ plan, const float* __restrict__ x,
                                                      float* __restrict__ y, long long N_) {
  spmv_tma_body<8>(plan, x, y, N_);
}

static const Builtin kHitsExp[] = {
    {"spmv_tma4", (const void*)k_spmv_tma4, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"spmv_tma8", (const void*)k_spmv_tma8, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"spmv_pad", (const void*)k_spmv_pad, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"spmv_pad_l2", (const void*)k_spmv_pad_l2, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"spmv_ws", (const void*)k_spmv_ws, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"spmv_hub4", (const void*)k_spmv_hub4, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 56 * 1024, nullptr, v_spmv_plan_kernel},
    {"spmv_hub2", (const void*)k_spmv_hub2, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 112 * 1024, nullptr, v_spmv_plan_kernel},
    {"spmv_hub1", (const void*)k_spmv_hub1, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 226 * 1024, nullptr, v_spmv_plan_kernel},
    {"spmv_pad2", (const void*)k_spmv_pad2, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"spmv_pad2b3", (const void*)k_spmv_pad2b3, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"spmv_nz", (const void*)k_spmv_nz, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"spmv_merge", (const void*)k_spmv, "const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE},
    {"spmv_plan", (const void*)k_spmv_plan, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE},
    {"spmv_plan_h", (const void*)k_spmv_plan_h, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE},
    {"spmv_sync", (const void*)k_spmv_sync, "const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE},
    {"spmv_x0s1", (const void*)k_spmv_x0s1, "const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE},
    {"spmv_x1s1", (const void*)k_spmv_x1s1, "const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE},
    {"spmv_as1", (const void*)k_spmv_as1, "const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE},
};
DAGRT_REGISTER_EXP(kHitsExp);

}  // namespace dagrt
