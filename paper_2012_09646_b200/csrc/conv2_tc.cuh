// DL second convolution on the tensor cores (§V-B,
// Fig. 6; reading R-DL): the pipeline building blocks (mbarriers,
// UMMA descriptors, TMA, TMEM access), the row-staged TMEM layout and the
// fp16-split kernel template k_conv2_h shared by the product instantiation
// (kernels_conv2.cu) and the experimental shapes (exp/conv2_variants.cu).
// The design notes are in kernels_conv2.cu.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "kcommon.cuh"

namespace dagrt {

// Pipeline trace points (compiled in only by tools/conv2_trace.cu, which
// defines C2_TRACE_ON and the buffer): SM clock of CTA 0 at each hand-off.
#ifdef C2_TRACE_ON
#define C2T(kind, i)                                                              \
  do {                                                                           \
    if (blockIdx.x == 0 && (i) < 64) g_c2trace[(kind) * 64 + (i)] = clock64();   \
  } while (0)
#else
#define C2T(kind, i) \
  do {               \
  } while (0)
#endif

namespace c2ws {

constexpr int kTaps = 9;
constexpr int kBox = 128 * 32;             // one tap: 128 pixels x 8 fp32, SWIZZLE_32B
constexpr int kStage = kTaps * kBox;       // 36 KB
constexpr int kBTap = 32 * 32;             // B per tap: 32 rows (16 hi + 16 lo) x 8 tf32
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccCols = 64;          // per buffer: acc32 (32) + acc16 (16), padded
constexpr uint32_t kLoCols = kTaps * 8;    // 72 tf32 columns of A_lo per buffer

// S TMA stages, NB TMEM buffers, SW split warps (a multiple of 4: SW/4 warps
// per TMEM lane quarter, sharing the 9 taps); warps 0-1 producer / MMA,
// 2..2+SW-1 split, then 4 epilogue warps
template <int S, int NB, int SW>
struct Cfg {
  static constexpr int kThreads = 32 * (2 + SW + 4);
  static constexpr uint32_t kLoBase = NB * kAccCols;
  static constexpr size_t smem() { return 1024 + (size_t)S * kStage + kTaps * kBTap + 8 * (2 * S + 3 * NB) + 16; }
  static_assert(kLoBase + NB * kLoCols <= kTmemCols, "TMEM budget");
  static_assert(SW % 4 == 0 && SW >= 4, "split warps per lane quarter");
};

// instruction descriptors: D f32, A/B tf32, K-major, M = 128
constexpr uint32_t idesc(uint32_t n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major no-swizzle descriptor (B: 8-row x 16-byte core matrices, LBO 128, SBO 256)
__device__ __forceinline__ uint64_t desc_plain(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
// K-major 32-byte-swizzle descriptor (the TMA box: 128 rows x 32 B, SBO 256)
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = su32(b);
  uint32_t done;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(done) : "r"(a), "r"(parity) : "memory");
  if (done) return;  // the common case: one probe, no guard bookkeeping
  for (uint32_t spins = 0; !done; ++spins) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
    if (spins > (1u << 30)) __trap();  // never hang the GPU on a protocol bug
  }
}
__device__ __forceinline__ void tma3d(uint32_t dst, const void* tmap, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
               : "memory");
}
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ uint32_t lo_bits(float x) {  // x - trunc_tf32(x), exact in fp32
  return __float_as_uint(x - __uint_as_float(__float_as_uint(x) & 0xffffe000u));
}

// Rows one TMA box delivers: 128, or ceil(W2/2) for inputs narrower than the
// 256-pixel box (the tensor map's box is clipped to the tensor, see the hook)
__device__ __forceinline__ int box_rows(int W2) { return W2 < 256 ? (W2 + 1) / 2 : 128; }

}  // namespace c2ws

// ---------------------------------------------------------------------------
// conv2, row-staged ("conv2_rows"): every input row is brought in ONCE.
//
// tools/tma_lab.py measured the 9-box-per-tile pattern above at 140 us for
// the TMA traffic alone (36 KB per 128-pixel tile from L2: ~30 B/clk/SM, the
// L2->SM ceiling), so the kernel cannot go below that however it overlaps.
// Here each CTA walks a contiguous run of output rows of one 128-pixel column
// block, so output row p needs only the two new input rows 2p, 2p+1 (row
// 2p-1 is the previous row's 2p+1): 16.5 KB per tile.  An input row segment
// (pixels 2 q0 - 2 .. 2 q0 + 255) is loaded as two planes of pixel PAIRS,
// parity 0 (even pixels) and parity 1 (odd pixels), by a 4-D tensor map
// {8 ch, 2 parities, W2/2 pairs, H2 rows}, box {8, 1, 129, 1} (no element
// stride, 32-byte swizzle -> conflict-free 16-byte reads); tap (a, b) of
// output pixel r is  b = 1: even[r],  b = 0: odd[r],  b = 2: odd[r + 1]
// (odd plane starting at pair q0 - 1).  Since these taps sit at a one-row
// offset the UMMA smem descriptors cannot express, the split warps write BOTH
// A_hi (13 low mantissa bits cleared) and A_lo into TMEM, and every MMA reads
// A from TMEM and only B from shared memory.  Rows are released to the TMA
// producer by the split warps as soon as no later tile needs them.
// Zero padding: rows and pairs outside the tensor come back as TMA zeros; for
// odd W2 the one pixel past the row end (parity 1 of the last pair) is zeroed
// by the split, and the input array needs 32 bytes of slack (validator).
namespace c2rows {
constexpr int kPlane = 129 * 32;                 // 4128 B: 129 pixels x 8 fp32
constexpr int kPlaneStride = 4352;               // rounded to 256 B (SW32 atoms)
constexpr int kSlot = 2 * kPlaneStride;          // one input row segment: even + odd planes
constexpr uint32_t kABase = 128;                 // TMEM: acc buffers at 0, 64; A buffers from 128
constexpr uint32_t kACols = 2 * c2ws::kLoCols;   // hi (72) + lo (72) per buffer

template <int R, int NB, int SW>
struct Cfg {
  static constexpr int kThreads = 32 * (2 + SW + 4);
  static constexpr size_t smem() {
    return 1024 + (size_t)R * kSlot + c2ws::kTaps * c2ws::kBTap + 8 * (2 * R + 3 * NB) + 16;
  }
  static_assert(kABase + NB * kACols <= c2ws::kTmemCols && NB * c2ws::kAccCols <= kABase, "TMEM budget");
  static_assert(SW % 4 == 0 && SW >= 4, "split warps per lane quarter");
};

// Tile t of CTA b (global order: column block major, output row minor).
struct Tile {
  int qb, p;
  bool chained;  // the previous tile of this CTA was (qb, p - 1): rows 2p-1 already loaded
};
__device__ __forceinline__ Tile tile_at(long long t, long long tprev, int H3) {
  Tile T;
  T.qb = (int)(t / H3);
  T.p = (int)(t % H3);
  T.chained = tprev >= 0 && t == tprev + 1 && T.p > 0;
  return T;
}
}  // namespace c2rows

// ---------------------------------------------------------------------------
// conv2 with ONE tensor-core instruction per tap ("conv2_h").
//
// tools/mma_lab.py: a tcgen05.mma with M = 128 costs ~47 cycles whatever
// N <= 64 (and kind), and the pipeline trace of conv2_ws (tools/conv2_trace.py)
// put its MMA thread on the critical path: 18 MMAs per tile (two 3xTF32
// chains) took ~1650 of the 2150 cycles per tile.  The split fp32 product
// x w = x_hi w_hi + x_lo w_hi + x_hi w_lo  (x_lo w_lo < 2^-22 |x w| dropped)
// needs only K = 16 per tap if the halves are fp16 (11-bit significands:
// x_hi = rn16(x), x_lo = rn16(x - x_hi), so x_hi + x_lo carries 22 bits like
// 3xTF32), so ONE kind::f16 MMA per tap does all three products:
//   A row (pixel) = [x_hi(c0..c7) | x_lo(c0..c7)]          (K = 16, in TMEM)
//   B rows n      = [w_hi(n, c0..c7) | w_hi(n, c0..c7)]    (n < 16)
//   B rows 16 + n = [w_lo(n, c0..c7) | 0]
//   D[:, n] + D[:, 16 + n] = x_hi w_hi + x_lo w_hi + x_hi w_lo   (fp32 accumulate)
// 9 MMAs per 128-pixel tile instead of 18, 8 TMEM columns of A per tap
// instead of 16, 32 accumulator columns instead of 48.  Numeric contract:
// |x|, |w| < 65504 (fp16 range; the DL activations are ReLU-conv-pool values
// bounded by 9 max|w1| < 4); halves below 2^-14 are fp16-subnormal, which
// costs at most 2^-25 absolute per element.  Rows are staged like
// conv2_rows (one pair-plane load per input row per column block).
namespace c2h {
constexpr uint32_t kACols = 9 * 8;  // A per buffer: 9 taps x 8 columns (16 fp16 per lane)
constexpr uint32_t kABase = 128;
constexpr int kBTap = 32 * 32;      // B per tap: 32 rows x 16 fp16

template <int R, int NB, int SW>
struct Cfg {
  static constexpr int kThreads = 32 * (2 + SW + 4);
  static constexpr size_t smem() {
    return 1024 + (size_t)R * c2rows::kSlot + 9 * kBTap + 8 * (2 * R + 3 * NB) + 16;
  }
  static_assert(NB * 32 <= (int)kABase && kABase + NB * kACols <= c2ws::kTmemCols, "TMEM budget");
  static_assert(SW % 4 == 0 && SW >= 4, "split warps per lane quarter");
};
// hi and lo halves of two fp32 values, packed two per 32-bit TMEM column (the
// first value in the low half): packed conversions (F2FP / HADD2.F32 on the
// ALU / FMA pipes) instead of scalar F2F on the quarter-rate XU pipe, which
// bounded the first version (275-330 us)
__device__ __forceinline__ void split_h2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
}  // namespace c2h

template <int R, int NB, int SW>
__global__ void __launch_bounds__(c2h::Cfg<R, NB, SW>::kThreads, 1)
    k_conv2_h(const CUtensorMap* __restrict__ tmap, const float* __restrict__ in, const float* __restrict__ w,
              float* __restrict__ out, int H2, int W2) {
  using namespace c2ws;
  using c2rows::kPlane;
  using c2rows::kPlaneStride;
  using c2rows::kSlot;
  using c2rows::Tile;
  using c2rows::tile_at;
  constexpr int kThreads = c2h::Cfg<R, NB, SW>::kThreads;
  constexpr uint32_t kABase = c2h::kABase, kACols = c2h::kACols;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* rows = sm;
  unsigned char* bt = rows + R * kSlot;                  // [9][32 rows x 32 B] fp16, interleaved
  uint64_t* full = reinterpret_cast<uint64_t*>(bt + 9 * c2h::kBTap);
  uint64_t* empty = full + R;
  uint64_t* loready = empty + R;
  uint64_t* mmadone = loready + NB;
  uint64_t* accempty = mmadone + NB;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accempty + NB);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  (void)in;

  // ---- B: per tap, row n < 16 = [w_hi | w_hi], row 16 + n = [w_lo | 0] (fp16, K-major)
  for (int i = t; i < 16 * 72; i += kThreads) {
    const int n = i / 72, r = i % 72, tap = r / 8, c = r % 8;
    const float x = w[i];
    const __half hi = __float2half_rn(x), lo = __float2half_rn(x - __half2float(hi));
    auto at = [&](int row, int k) -> __half* {  // element k (0..15) of B row `row`
      return reinterpret_cast<__half*>(bt + tap * c2h::kBTap + (row & 7) * 16 + (row >> 3) * 256 + (k >> 3) * 128 +
                                       (k & 7) * 2);
    };
    *at(n, c) = hi;
    *at(n, 8 + c) = hi;
    *at(16 + n, c) = lo;
    *at(16 + n, 8 + c) = __float2half_rn(0.f);
  }
  if (t == 0) {
    for (int q = 0; q < R; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, SW);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(loready + b, SW);
      mbar_init(mmadone + b, 1);
      mbar_init(accempty + b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (tmap) asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;

  const int H3 = (H2 + 1) / 2, W3 = (W2 + 1) / 2;
  const int nqb = (W3 + 127) / 128;
  const long long ntiles = (long long)H3 * nqb;
  const long long per = (ntiles + gridDim.x - 1) / gridDim.x;
  const long long tb = (long long)blockIdx.x * per, te = min(ntiles, tb + per);
  const int nmine = te > tb ? (int)(te - tb) : 0;
  // (qb, p) of the CTA's first tile; later tiles advance p, wrapping to the next column block
  const int qb0 = (int)(tb / H3), p0 = (int)(tb % H3);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t tx = 2u * kPlane;
      int rseq = 0, qb = qb0, p = p0;
      for (int i = 0; i < nmine; ++i) {
        const bool chained = i > 0 && p > 0;
        const int q0 = qb * 128;
        for (int a = chained ? 1 : 0; a < 3; ++a, ++rseq) {
          const int slot = rseq % R;
          mbar_wait(empty + slot, (uint32_t)(((rseq / R) & 1) ^ 1));
          if (a == 2) C2T(0, i);
          const uint32_t bar = su32(full + slot);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
          const int y = 2 * p + a - 1;
          unsigned char* dst = rows + slot * kSlot;
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
              ::"r"(su32(dst)), "l"(tmap), "r"(0), "r"(0), "r"(q0), "r"(y), "r"(bar) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
              ::"r"(su32(dst + kPlaneStride)), "l"(tmap), "r"(0), "r"(1), "r"(q0 - 1), "r"(y), "r"(bar) : "memory");
        }
        C2T(1, i);
        if (++p == H3) { p = 0; ++qb; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kId = (1u << 4) | (0u << 7) | (0u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
      for (int i = 0; i < nmine; ++i) {
        const int b = i % NB;
        const uint32_t pb = (uint32_t)((i / NB) & 1);
        mbar_wait(loready + b, pb);
        C2T(2, i);
        mbar_wait(accempty + b, pb ^ 1);
        C2T(3, i);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + b * 32, a = tmem + kABase + b * kACols;
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const uint64_t bd = desc_plain(su32(bt + tap * c2h::kBTap));
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(d), "r"(a + tap * 8),
                       "l"(bd), "r"(kId), "r"((uint32_t)(tap > 0)));
        }
        commit(mmadone + b);
        C2T(4, i);
      }
    }
  } else if (warp < 2 + SW) {
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const int part = (warp - 2) / 4;
    constexpr int kShares = SW / 4;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int rseq = 0, qb = qb0, p = p0;
    for (int i = 0; i < nmine; ++i) {
      const bool chained = i > 0 && p > 0;
      const int nq = p + 1 == H3 ? 0 : p + 1;  // the next tile chains unless it wraps or is not ours
      const bool next_chained = i + 1 < nmine && nq > 0;
      const int s0 = chained ? rseq - 1 : rseq;
      const int b = i % NB;
      mbar_wait(mmadone + b, (uint32_t)(((i / NB) & 1) ^ 1));
      if (warp == 2 && lane == 0) C2T(6, i);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t abuf = tmem + lane_off + kABase + b * kACols;
      const bool edge = 2 * (qb * 128 + r) + 1 >= W2;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        // only the rows holding one of this part's taps are waited for and
        // read (each try_wait costs ~100+ cycles even when the row is ready:
        // ncu put a quarter of the split warps' samples on these waits)
        if ((3 * a * kShares) / 9 != part && ((3 * a + 1) * kShares) / 9 != part && ((3 * a + 2) * kShares) / 9 != part)
          continue;
        const int rs = s0 + a;
        const int slot = rs % R;
        mbar_wait(full + slot, (uint32_t)((rs / R) & 1));
        if (a == 2 && warp == 2 && lane == 0) C2T(5, i);
        const unsigned char* ev = rows + slot * kSlot;
        const unsigned char* od = ev + kPlaneStride;
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          const int tap = a * 3 + bb;
          if ((tap * kShares) / 9 != part) continue;
          const int row = bb == 2 ? r + 1 : r;
          const unsigned char* pl = (bb == 1 ? ev : od) + 32 * row;
          const int sw = (row >> 2) & 1;
          float4 x0 = *reinterpret_cast<const float4*>(pl + 16 * sw);
          float4 x1 = *reinterpret_cast<const float4*>(pl + 16 * (sw ^ 1));
          if (bb == 2 && edge) x0 = x1 = make_float4(0.f, 0.f, 0.f, 0.f);
          uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
          c2h::split_h2(x0.x, x0.y, h0, l0);
          c2h::split_h2(x0.z, x0.w, h1, l1);
          c2h::split_h2(x1.x, x1.y, h2, l2);
          c2h::split_h2(x1.z, x1.w, h3, l3);
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(abuf + tap * 8),
                       "r"(h0), "r"(h1), "r"(h2), "r"(h3), "r"(l0), "r"(l1), "r"(l2), "r"(l3)
                       : "memory");
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (warp == 2 && lane == 0) C2T(7, i);
      if (lane == 0) {
        mbar_arrive(loready + b);
        mbar_arrive(empty + (s0 % R));
        mbar_arrive(empty + ((s0 + 1) % R));
        if (!next_chained) mbar_arrive(empty + ((s0 + 2) % R));
      }
      rseq += chained ? 2 : 3;
      if (++p == H3) { p = 0; ++qb; }
    }
  } else {
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int qb = qb0, p = p0;
    for (int i = 0; i < nmine; ++i) {
      const int b = i % NB;
      mbar_wait(mmadone + b, (uint32_t)((i / NB) & 1));
      if (warp == 2 + SW && lane == 0) C2T(8, i);
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t h[16], l[16];
      const uint32_t d = tmem + lane_off + b * 32;
      ld16(d, h);
      ld16(d + 16, l);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty + b);
      const int q = qb * 128 + r;
      if (q < W3) {
        float4* dst = reinterpret_cast<float4*>(out + ((size_t)p * W3 + q) * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = fmaxf(__uint_as_float(h[4 * k + j]) + __uint_as_float(l[4 * k + j]), 0.f);
          dst[k] = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
      if (warp == 2 + SW && lane == 0) C2T(9, i);
      if (++p == H3) { p = 0; ++qb; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}


// conv2_hs: k_conv2_h with the A operand in SHARED memory (the canonical
// K-major no-swizzle layout, one 4 KB block per tap) instead of TMEM.  The
// pipeline trace of the product (tools/conv2h_trace.py) has the split stage
// on the critical path at ~1200 cycles per tile and 9 MMAs taking ~800
// cycles to issue (vs ~47 cycles each in tools/mma_lab.py) while more split
// warps make it slower: split stores into TMEM and the MMAs' A reads from
// TMEM contend.  Here the split writes A with two 16-byte shared stores per
// tap and pixel and the MMAs read A and B from shared memory (SS).
namespace c2hs {
constexpr int kATap = 128 * 32;  // A per tap: 128 rows x 16 fp16
template <int R, int NB, int SW>
struct Cfg {
  static constexpr int kThreads = 32 * (2 + SW + 4);
  static constexpr size_t smem() {
    return 1024 + (size_t)R * c2rows::kSlot + 9 * c2h::kBTap + (size_t)NB * 9 * kATap + 8 * (2 * R + 3 * NB) + 16;
  }
  static_assert(NB * 32 <= (int)c2h::kABase, "TMEM budget");
  static_assert(SW % 4 == 0 && SW >= 4, "split warps per lane quarter");
  static_assert(smem() <= 227 * 1024, "shared memory budget");
};
}  // namespace c2hs

template <int R, int NB, int SW>
__global__ void __launch_bounds__(c2hs::Cfg<R, NB, SW>::kThreads, 1)
    k_conv2_hs(const CUtensorMap* __restrict__ tmap, const float* __restrict__ in, const float* __restrict__ w,
              float* __restrict__ out, int H2, int W2) {
  using namespace c2ws;
  using c2rows::kPlane;
  using c2rows::kPlaneStride;
  using c2rows::kSlot;
  using c2rows::Tile;
  using c2rows::tile_at;
  constexpr int kThreads = c2hs::Cfg<R, NB, SW>::kThreads;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* rows = sm;
  unsigned char* bt = rows + R * kSlot;                  // [9][32 rows x 32 B] fp16, interleaved
  unsigned char* as = bt + 9 * c2h::kBTap;               // A: [NB][9 taps][128 rows x 32 B] fp16, interleaved
  uint64_t* full = reinterpret_cast<uint64_t*>(as + NB * 9 * c2hs::kATap);
  uint64_t* empty = full + R;
  uint64_t* loready = empty + R;
  uint64_t* mmadone = loready + NB;
  uint64_t* accempty = mmadone + NB;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accempty + NB);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  (void)in;

  // ---- B: per tap, row n < 16 = [w_hi | w_hi], row 16 + n = [w_lo | 0] (fp16, K-major)
  for (int i = t; i < 16 * 72; i += kThreads) {
    const int n = i / 72, r = i % 72, tap = r / 8, c = r % 8;
    const float x = w[i];
    const __half hi = __float2half_rn(x), lo = __float2half_rn(x - __half2float(hi));
    auto at = [&](int row, int k) -> __half* {  // element k (0..15) of B row `row`
      return reinterpret_cast<__half*>(bt + tap * c2h::kBTap + (row & 7) * 16 + (row >> 3) * 256 + (k >> 3) * 128 +
                                       (k & 7) * 2);
    };
    *at(n, c) = hi;
    *at(n, 8 + c) = hi;
    *at(16 + n, c) = lo;
    *at(16 + n, 8 + c) = __float2half_rn(0.f);
  }
  if (t == 0) {
    for (int q = 0; q < R; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, SW);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(loready + b, SW);
      mbar_init(mmadone + b, 1);
      mbar_init(accempty + b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (tmap) asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;

  const int H3 = (H2 + 1) / 2, W3 = (W2 + 1) / 2;
  const int nqb = (W3 + 127) / 128;
  const long long ntiles = (long long)H3 * nqb;
  const long long per = (ntiles + gridDim.x - 1) / gridDim.x;
  const long long tb = (long long)blockIdx.x * per, te = min(ntiles, tb + per);
  const int nmine = te > tb ? (int)(te - tb) : 0;
  // (qb, p) of the CTA's first tile; later tiles advance p, wrapping to the next column block
  const int qb0 = (int)(tb / H3), p0 = (int)(tb % H3);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t tx = 2u * kPlane;
      int rseq = 0, qb = qb0, p = p0;
      for (int i = 0; i < nmine; ++i) {
        const bool chained = i > 0 && p > 0;
        const int q0 = qb * 128;
        for (int a = chained ? 1 : 0; a < 3; ++a, ++rseq) {
          const int slot = rseq % R;
          mbar_wait(empty + slot, (uint32_t)(((rseq / R) & 1) ^ 1));
          if (a == 2) C2T(0, i);
          const uint32_t bar = su32(full + slot);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
          const int y = 2 * p + a - 1;
          unsigned char* dst = rows + slot * kSlot;
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
              ::"r"(su32(dst)), "l"(tmap), "r"(0), "r"(0), "r"(q0), "r"(y), "r"(bar) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
              ::"r"(su32(dst + kPlaneStride)), "l"(tmap), "r"(0), "r"(1), "r"(q0 - 1), "r"(y), "r"(bar) : "memory");
        }
        C2T(1, i);
        if (++p == H3) { p = 0; ++qb; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kId = (1u << 4) | (0u << 7) | (0u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
      for (int i = 0; i < nmine; ++i) {
        const int b = i % NB;
        const uint32_t pb = (uint32_t)((i / NB) & 1);
        mbar_wait(loready + b, pb);
        C2T(2, i);
        mbar_wait(accempty + b, pb ^ 1);
        C2T(3, i);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + b * 32;
        const uint32_t a = su32(as + b * 9 * c2hs::kATap);
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const uint64_t bd = desc_plain(su32(bt + tap * c2h::kBTap));
          const uint64_t ad = desc_plain(a + tap * c2hs::kATap);
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d), "l"(ad),
                       "l"(bd), "r"(kId), "r"((uint32_t)(tap > 0)));
        }
        commit(mmadone + b);
        C2T(4, i);
      }
    }
  } else if (warp < 2 + SW) {
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const int part = (warp - 2) / 4;
    constexpr int kShares = SW / 4;
    int rseq = 0, qb = qb0, p = p0;
    for (int i = 0; i < nmine; ++i) {
      const bool chained = i > 0 && p > 0;
      const int nq = p + 1 == H3 ? 0 : p + 1;  // the next tile chains unless it wraps or is not ours
      const bool next_chained = i + 1 < nmine && nq > 0;
      const int s0 = chained ? rseq - 1 : rseq;
      const int b = i % NB;
      mbar_wait(mmadone + b, (uint32_t)(((i / NB) & 1) ^ 1));
      if (warp == 2 && lane == 0) C2T(6, i);
      asm volatile("tcgen05.fence::after_thread_sync;");
      unsigned char* abuf = as + b * 9 * c2hs::kATap + (r & 7) * 16 + (r >> 3) * 256;  // this pixel's A row
      const bool edge = 2 * (qb * 128 + r) + 1 >= W2;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int rs = s0 + a;
        const int slot = rs % R;
        mbar_wait(full + slot, (uint32_t)((rs / R) & 1));
        if (a == 2 && warp == 2 && lane == 0) C2T(5, i);
        const unsigned char* ev = rows + slot * kSlot;
        const unsigned char* od = ev + kPlaneStride;
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          const int tap = a * 3 + bb;
          if ((tap * kShares) / 9 != part) continue;
          const int row = bb == 2 ? r + 1 : r;
          const unsigned char* pl = (bb == 1 ? ev : od) + 32 * row;
          const int sw = (row >> 2) & 1;
          float4 x0 = *reinterpret_cast<const float4*>(pl + 16 * sw);
          float4 x1 = *reinterpret_cast<const float4*>(pl + 16 * (sw ^ 1));
          if (bb == 2 && edge) x0 = x1 = make_float4(0.f, 0.f, 0.f, 0.f);
          uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
          c2h::split_h2(x0.x, x0.y, h0, l0);
          c2h::split_h2(x0.z, x0.w, h1, l1);
          c2h::split_h2(x1.x, x1.y, h2, l2);
          c2h::split_h2(x1.z, x1.w, h3, l3);
          *reinterpret_cast<uint4*>(abuf + tap * c2hs::kATap) = make_uint4(h0, h1, h2, h3);        // k 0..7: hi
          *reinterpret_cast<uint4*>(abuf + tap * c2hs::kATap + 128) = make_uint4(l0, l1, l2, l3);  // k 8..15: lo
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy A writes -> the MMA
      __syncwarp();
      if (warp == 2 && lane == 0) C2T(7, i);
      if (lane == 0) {
        mbar_arrive(loready + b);
        mbar_arrive(empty + (s0 % R));
        mbar_arrive(empty + ((s0 + 1) % R));
        if (!next_chained) mbar_arrive(empty + ((s0 + 2) % R));
      }
      rseq += chained ? 2 : 3;
      if (++p == H3) { p = 0; ++qb; }
    }
  } else {
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int qb = qb0, p = p0;
    for (int i = 0; i < nmine; ++i) {
      const int b = i % NB;
      mbar_wait(mmadone + b, (uint32_t)((i / NB) & 1));
      if (warp == 2 + SW && lane == 0) C2T(8, i);
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t h[16], l[16];
      const uint32_t d = tmem + lane_off + b * 32;
      ld16(d, h);
      ld16(d + 16, l);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty + b);
      const int q = qb * 128 + r;
      if (q < W3) {
        float4* dst = reinterpret_cast<float4*>(out + ((size_t)p * W3 + q) * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = fmaxf(__uint_as_float(h[4 * k + j]) + __uint_as_float(l[4 * k + j]), 0.f);
          dst[k] = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
      if (warp == 2 + SW && lane == 0) C2T(9, i);
      if (++p == H3) { p = 0; ++qb; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}


// Pre-launch hook of the row-staged kernels (kernels_conv2.cu): the 4-D
// pair-plane tensor map of the input, cached per (device, pointer, shape).
int conv2_rows_prelaunch(const uint64_t* vals, int nargs, void** extra);

// launch contract (dagrt_launch validates it before the pre-launch hook)
static inline const char* v_conv2_launch(const LaunchCheck& L, unsigned threads, unsigned smem_min) {  // in, w, out, H2, W2
  const int H2 = L.i32(3), W2 = L.i32(4);
  if (H2 < 0 || W2 < 0) return "negative size";
  const uint64_t H3 = (H2 + 1) / 2, W3 = (W2 + 1) / 2;
  if (!fits(L, 0, 32ull * H2 * W2) || !fits(L, 1, 4 * 16 * 72) || !fits(L, 2, 64 * H3 * W3))
    return "in (32 H2 W2), w (4608) or out (64 H3 W3) too small";
  if (L.vals[0] % 16) return "the input must be 16-byte aligned (TMA)";
  if (L.block[0] != threads || L.block[1] != 1 || L.block[2] != 1) return "wrong block size for this kernel";
  if (L.smem < smem_min) return "dynamic shared memory below the kernel's layout";
  return nullptr;
}
template <int R, int NB, int SW>
static const char* v_conv2_h(const LaunchCheck& L) {
  using C = c2h::Cfg<R, NB, SW>;
  if (const char* e = v_conv2_launch(L, C::kThreads, (unsigned)C::smem())) return e;
  if ((L.i32(4) & 1) && !fits(L, 0, 32ull * L.i32(3) * L.i32(4) + 32)) return "odd W2 needs 32 bytes of input slack";
  return nullptr;
}
template <int R, int NB, int SW>
static const char* v_conv2_hs(const LaunchCheck& L) {
  using C = c2hs::Cfg<R, NB, SW>;
  if (const char* e = v_conv2_launch(L, C::kThreads, (unsigned)C::smem())) return e;
  if ((L.i32(4) & 1) && !fits(L, 0, 32ull * L.i32(3) * L.i32(4) + 32)) return "odd W2 needs 32 bytes of input slack";
  return nullptr;
}
#define C2HS(NAME, R, NB, SW)                                                                            \
  {NAME, (const void*)k_conv2_hs<R, NB, SW>, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, \
   (int)c2hs::Cfg<R, NB, SW>::smem(), conv2_rows_prelaunch, v_conv2_hs<R, NB, SW>}
#define C2H(NAME, R, NB, SW)                                                                            \
  {NAME, (const void*)k_conv2_h<R, NB, SW>, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, \
   (int)c2h::Cfg<R, NB, SW>::smem(), conv2_rows_prelaunch, v_conv2_h<R, NB, SW>}

}  // namespace dagrt
