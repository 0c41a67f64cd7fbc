// TMEM laboratory (tools only): does tcgen05.mma.kind::tf32 with the A
// operand in TENSOR MEMORY compute D = A B for M = 128, N = 16, K = 8 per
// instruction, with A row i = TMEM lane i and its K elements in consecutive
// 32-bit columns (written by each thread with tcgen05.st 32x32b)?  9 taps
// (K = 72) accumulate into one 16-column accumulator.  MODE 0: A in shared
// memory (the layout the conv2 kernels use, known good); MODE 1: A in TMEM.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

template <int MODE>
__global__ void __launch_bounds__(128, 1) k_tmem_mma(const float* __restrict__ A, const float* __restrict__ B,
                                                     float* __restrict__ D) {
  __shared__ __align__(1024) unsigned char sb[9 * 512];
  __shared__ __align__(1024) unsigned char sa[9 * 4096];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 16 * 72; i += 128) {  // B[k][tap*8 + c], K-major no-swizzle core matrices
    const int k = i / 72, r = i % 72, tap = r / 8, c = r % 8;
    *reinterpret_cast<float*>(sb + tap * 512 + (k & 7) * 16 + (k >> 3) * 256 + (c >> 2) * 128 + (c & 3) * 4) = B[i];
  }
  if (MODE == 0)
    for (int tap = 0; tap < 9; ++tap)
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<float*>(sa + tap * 4096 + (t & 7) * 16 + (t >> 3) * 256 + (c >> 2) * 128 + (c & 3) * 4) =
            A[t * 72 + tap * 8 + c];
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (MODE == 1) {
    for (int tap = 0; tap < 9; ++tap) {
      uint32_t r[8];
      for (int c = 0; c < 8; ++c) r[c] = __float_as_uint(A[t * 72 + tap * 8 + c]);
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 32 + tap * 8;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(r[0]),
                   "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                   : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    for (int tap = 0; tap < 9; ++tap) {
      const uint64_t bd = umma_desc(smem_u32(sb + tap * 512), 128, 256);
      const uint32_t acc = tap > 0;
      if (MODE == 0) {
        const uint64_t ad = umma_desc(smem_u32(sa + tap * 4096), 128, 256);
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
      } else {
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }" ::"r"(tmem),
                     "r"(tmem + 32 + tap * 8), "l"(bd), "r"(kIdesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int k = 0; k < 16; ++k) D[t * 16 + k] = __uint_as_float(r[k]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

}  // namespace

// MODE 2: kind::f16 with fp16 operands, A (128 x 64 fp16) in TMEM, two fp16
// per 32-bit column (element 2j in the low half), 4 MMAs of K = 16; B (16 x 64
// fp16) in shared memory, K-major no swizzle (32 B per row per MMA).
__global__ void __launch_bounds__(128, 1) k_tmem_f16(const __half* __restrict__ A, const __half* __restrict__ B,
                                                     float* __restrict__ D) {
  __shared__ __align__(1024) unsigned char sb[4 * 512];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 16 * 64; i += 128) {  // B[n][k]: MMA q = k / 16, kk = k % 16
    const int n = i / 64, k = i % 64, q = k / 16, kk = k % 16;
    *reinterpret_cast<__half*>(sb + q * 512 + (n & 7) * 16 + (n >> 3) * 256 + (kk >> 3) * 128 + (kk & 7) * 2) = B[i];
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  for (int q = 0; q < 4; ++q) {
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) {
      const __half lo = A[t * 64 + q * 16 + 2 * j], hi = A[t * 64 + q * 16 + 2 * j + 1];
      r[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 32 + q * 8;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    const uint32_t idf16 = (1u << 4) | (0u << 7) | (0u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
    for (int q = 0; q < 4; ++q) {
      const uint64_t bd = umma_desc(smem_u32(sb + q * 512), 128, 256);
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(tmem),
                   "r"(tmem + 32 + q * 8), "l"(bd), "r"(idf16), "r"((uint32_t)(q > 0)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int k = 0; k < 16; ++k) D[t * 16 + k] = __uint_as_float(r[k]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

extern "C" int tmem_lab_f16(const void* A, const void* B, float* D) {
  k_tmem_f16<<<1, 128>>>((const __half*)A, (const __half*)B, D);
  return (int)cudaDeviceSynchronize();
}

extern "C" int tmem_lab(int mode, const float* A, const float* B, float* D) {
  if (mode == 0) k_tmem_mma<0><<<1, 128>>>(A, B, D);
  else k_tmem_mma<1><<<1, 128>>>(A, B, D);
  return (int)cudaDeviceSynchronize();
}
