// DL second convolution, round 2: warp-specialised TMA -> tcgen05 pipeline
// with the A_lo operand of 3xTF32 in TENSOR MEMORY.
//
// conv2 (§V-B, Fig. 6; reading R-DL):
//   c2[p, q, n] = ReLU(sum_{a,b,c} W2[n, a, b, c] p[2p+a-1, 2q+b-1, c]),
// an implicit GEMM per 128-pixel tile: M = 128 output pixels (one output row
// segment), N = 16 channels, K = 72 = 9 taps x 8 input channels.  fp32 to
// the north_star's 1e-4 needs 3xTF32:  D = A_hi B_hi + A_hi B_lo + A_lo B_hi.
//
// Round-1 product (k_conv2_tmang, kernels_conv_tc.cu) ran 285 us per branch:
// three consumer groups of 128 threads, each with ONE TMA stage, serialised
// TMA wait -> split -> MMA -> wait -> epilogue, so ~3 tiles were in flight per
// SM and the long TMA/MMA/epilogue latencies were exposed; its A_lo tiles
// also went through shared memory twice (written by threads, read by the
// tensor core).  Here every role runs concurrently on different tiles:
//
//   warp 0      TMA producer: 9 stride-2 boxes {8 ch, 128 px, 1 row} per tile
//               (tap (a,b) = pixels 2q+b-1 of input row 2p+a-1; zero padding
//               by TMA out-of-bounds fill) into an S-stage ring (36 KB/stage);
//   warps 2-5   split: each thread (= TMEM lane = output pixel) reads its 9
//               taps from the swizzled box, forms lo = x - trunc_tf32(x) and
//               stores it into TMEM (tcgen05.st) -- A_lo never touches smem;
//   warp 1      MMA issuer (one thread): per tap an N=32 MMA A_hi x [B_hi|B_lo]
//               with A_hi = the raw box in smem (the tensor core truncates
//               fp32 to tf32, pinned by test_tensor_core_truncates_fp32_to_tf32)
//               and an N=16 MMA A_lo(TMEM) x B_hi; commits release the stage
//               and hand the accumulators to the epilogue;
//   warps 6-9   epilogue: tcgen05.ld of the 48 accumulator columns, sum of the
//               three products, ReLU, 64 B per pixel to global memory.
// NB accumulator / A_lo buffers in TMEM (512 columns) decouple MMA, split and
// epilogue; mbarriers carry every hand-off (full/empty per stage, lo-ready /
// mma-done / acc-empty per buffer).  A-from-TMEM kind::tf32 semantics are
// pinned by tools/tmem_lab.py (matches A-from-smem bit for bit).
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "kcommon.cuh"

namespace dagrt {

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
  uint32_t done = 0;
  long long spins = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
    if (++spins > (1ll << 30)) __trap();  // never hang the GPU on a protocol bug
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

template <int S, int NB, int SW>
__global__ void __launch_bounds__(c2ws::Cfg<S, NB, SW>::kThreads, 1)
    k_conv2_ws(const CUtensorMap* __restrict__ tmap, const float* __restrict__ in, const float* __restrict__ w,
               float* __restrict__ out, int H2, int W2) {
  using namespace c2ws;
  constexpr int kStages = S, kBufs = NB, kThreads = Cfg<S, NB, SW>::kThreads;
  constexpr uint32_t kLoBase = Cfg<S, NB, SW>::kLoBase;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* raw = sm;                               // [S][9][128 x 32 B] SW32
  unsigned char* bt = raw + kStages * kStage;            // [9][32 rows x 32 B] interleaved
  uint64_t* full = reinterpret_cast<uint64_t*>(bt + kTaps * kBTap);
  uint64_t* empty = full + kStages;
  uint64_t* loready = empty + kStages;
  uint64_t* mmadone = loready + kBufs;
  uint64_t* accempty = mmadone + kBufs;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accempty + kBufs);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  (void)in;

  // ---- setup: B = [W2_hi ; W2_lo] per tap (32 x 8 tf32), barriers, TMEM
  for (int i = t; i < 16 * 72; i += kThreads) {
    const int k = i / 72, r = i % 72, tap = r / 8, c = r % 8;
    const float x = w[i];
    uint32_t hi;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
    uint32_t lo;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(x - __uint_as_float(hi)));
    auto off = [&](int row) { return tap * kBTap + (row & 7) * 16 + (row >> 3) * 256 + (c >> 2) * 128 + (c & 3) * 4; };
    *reinterpret_cast<uint32_t*>(bt + off(k)) = hi;
    *reinterpret_cast<uint32_t*>(bt + off(16 + k)) = lo;
  }
  if (t == 0) {
    for (int q = 0; q < kStages; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, 1);
    }
    for (int b = 0; b < kBufs; ++b) {
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
  const long long G = gridDim.x;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / G + 1) : 0;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      const uint32_t tx = 9u * 32u * (uint32_t)box_rows(W2);
      for (int i = 0; i < nmine; ++i) {
        const long long tile = blockIdx.x + (long long)i * G;
        const int s = i % kStages;
        mbar_wait(empty + s, (uint32_t)(((i / kStages) & 1) ^ 1));
        const int p = (int)(tile / nqb), q0 = (int)(tile % nqb) * 128;
        const uint32_t bar = su32(full + s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            tma3d(su32(raw + s * kStage + (a * 3 + b) * kBox), tmap, 0, 2 * q0 + b - 1, 2 * p + a - 1, bar);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      for (int i = 0; i < nmine; ++i) {
        const int s = i % kStages, b = i % kBufs;
        const uint32_t pb = (uint32_t)((i / kBufs) & 1);
        mbar_wait(loready + b, pb);       // A_lo in TMEM (and the stage's TMA data seen by the split)
        mbar_wait(accempty + b, pb ^ 1);  // the epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d32 = tmem + b * kAccCols, d16 = d32 + 32, alo = tmem + kLoBase + b * kLoCols;
#pragma unroll
        for (int tap = 0; tap < kTaps; ++tap) {
          const uint64_t ah = desc_sw32(su32(raw + s * kStage + tap * kBox));
          const uint64_t bd = desc_plain(su32(bt + tap * kBTap));
          const uint32_t acc = tap > 0;
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(d32), "l"(ah), "l"(bd),
                       "r"(idesc(32)), "r"(acc));
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }" ::"r"(d16),
                       "r"(alo + tap * 8), "l"(bd), "r"(idesc(16)), "r"(acc));
        }
        commit(empty + s);    // stage s may be refilled
        commit(mmadone + b);  // accumulators ready; A_lo buffer free
      }
    }
  } else if (warp < 2 + SW) {
    // ---------------- split: lo = x - trunc_tf32(x) -> TMEM (lane = pixel row)
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const int part = (warp - 2) / 4;  // which share of the taps (SW / 4 shares)
    constexpr int kShares = SW / 4;
    constexpr int kPer = (kTaps + kShares - 1) / kShares;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int i = 0; i < nmine; ++i) {
      const int s = i % kStages, b = i % kBufs;
      mbar_wait(full + s, (uint32_t)((i / kStages) & 1));
      mbar_wait(mmadone + b, (uint32_t)(((i / kBufs) & 1) ^ 1));  // A_lo buffer b consumed
      asm volatile("tcgen05.fence::after_thread_sync;");
      const unsigned char* rs = raw + s * kStage + 32 * r;
      const int sw = (r >> 2) & 1;  // 32-byte swizzle: chunk c of row r at 16 (c ^ ((r >> 2) & 1))
      const uint32_t alo = tmem + lane_off + kLoBase + b * kLoCols;
#pragma unroll
      for (int tt = 0; tt < kPer; ++tt) {
        const int tap = part * kPer + tt;
        if (tap >= kTaps) break;
        const float4 x0 = *reinterpret_cast<const float4*>(rs + tap * kBox + 16 * sw);
        const float4 x1 = *reinterpret_cast<const float4*>(rs + tap * kBox + 16 * (sw ^ 1));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(alo + tap * 8),
                     "r"(lo_bits(x0.x)), "r"(lo_bits(x0.y)), "r"(lo_bits(x0.z)), "r"(lo_bits(x0.w)),
                     "r"(lo_bits(x1.x)), "r"(lo_bits(x1.y)), "r"(lo_bits(x1.z)), "r"(lo_bits(x1.w))
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(loready + b);
    }
  } else {
    // ---------------- epilogue: ReLU(acc_hh + acc_hl + acc_lh), 64 B per pixel
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int i = 0; i < nmine; ++i) {
      const long long tile = blockIdx.x + (long long)i * G;
      const int b = i % kBufs;
      mbar_wait(mmadone + b, (uint32_t)((i / kBufs) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t h[16], l[16], m[16];
      const uint32_t d = tmem + lane_off + b * kAccCols;
      ld16(d, h);
      ld16(d + 16, l);
      ld16(d + 32, m);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty + b);
      const int p = (int)(tile / nqb), q = (int)(tile % nqb) * 128 + r;
      if (q < W3) {
        float4* dst = reinterpret_cast<float4*>(out + ((size_t)p * W3 + q) * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int n = 4 * k + j;
            v[j] = fmaxf(__uint_as_float(h[n]) + __uint_as_float(l[n]) + __uint_as_float(m[n]), 0.f);
          }
          dst[k] = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

int conv2_tma_prelaunch(const uint64_t* vals, int nargs, void** extra);  // kernels_conv_tc.cu

// launch contract (dagrt_launch validates it before the pre-launch hook)
static const char* v_conv2_tc(const LaunchCheck& L, unsigned threads, unsigned smem_min) {  // in, w, out, H2, W2
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
template <int S, int NB, int SW>
static const char* v_conv2_ws(const LaunchCheck& L) {
  using C = c2ws::Cfg<S, NB, SW>;
  return v_conv2_tc(L, C::kThreads, (unsigned)C::smem());
}

#define C2WS(NAME, S, NB, SW)                                                                            \
  {NAME, (const void*)k_conv2_ws<S, NB, SW>, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, \
   (int)c2ws::Cfg<S, NB, SW>::smem(), conv2_tma_prelaunch, v_conv2_ws<S, NB, SW>}
static const Builtin kConv2Ws[] = {
    // warp-specialised TMA -> tcgen05 conv2 with A_lo in TMEM, 148 CTAs:
    // S TMA stages, NB TMEM buffers, SW split warps (threads 32 (6 + SW),
    // c2ws::Cfg<S, NB, SW>::smem() bytes of dynamic shared memory)
    C2WS("conv2_ws", 4, 2, 4),
    C2WS("conv2_ws6", 6, 2, 4),
    C2WS("conv2_ws6s8", 6, 2, 8),
    C2WS("conv2_ws6b3", 6, 3, 4),
    C2WS("conv2_ws5s8b3", 5, 3, 8),
};
DAGRT_REGISTER_BUILTINS(kConv2Ws);

}  // namespace dagrt
