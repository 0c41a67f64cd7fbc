// tcgen05.mma cost laboratory (tools only): cycles per MMA instruction for
// M = 128 and N = 16..256, kind::tf32 (K = 8) and kind::f16 (bf16, K = 16),
// with A from shared memory (SS) or from tensor memory (TS).  One thread
// issues `reps` dependent MMAs into one accumulator, then a commit; the SM
// clock is read before the first issue, after the last issue and when the
// commit's mbarrier completes.  The operands' contents are irrelevant here.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_plain(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
// kind: 0 tf32 (A/B fmt 2), 1 bf16 (A/B fmt 1 in the f16 kind)
__device__ __forceinline__ uint32_t idesc(int kind, uint32_t n) {
  const uint32_t ab = kind == 0 ? 2u : 1u;
  return (1u << 4) | (ab << 7) | (ab << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

template <int KIND, int TS>
__global__ void __launch_bounds__(128, 1) k_mma(int n, int reps, long long* out) {
  __shared__ __align__(1024) unsigned char a[128 * 64];   // 128 rows x 32 B (one K step)
  __shared__ __align__(1024) unsigned char b[256 * 64];   // up to 256 rows x 32 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 64 / 4; i += 128) reinterpret_cast<float*>(a)[i] = 0.f;
  for (int i = t; i < 256 * 64 / 4; i += 128) reinterpret_cast<float*>(b)[i] = 0.f;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (t == 0) {
    const uint64_t ad = desc_plain(su32(a)), bd = desc_plain(su32(b));
    const uint32_t id = idesc(KIND, (uint32_t)n);
    long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t acc = r > 0;
      if (KIND == 0) {
        if (TS)
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }"
                       ::"r"(tmem), "r"(tmem + 256), "l"(bd), "r"(id), "r"(acc));
        else
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                       ::"r"(tmem), "l"(ad), "l"(bd), "r"(id), "r"(acc));
      } else {
        if (TS)
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
                       ::"r"(tmem), "r"(tmem + 256), "l"(bd), "r"(id), "r"(acc));
        else
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                       ::"r"(tmem), "l"(ad), "l"(bd), "r"(id), "r"(acc));
      }
    }
    long long c1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&bar)), "r"(0) : "memory");
    long long c2 = clock64();
    out[0] = c1 - c0;
    out[1] = c2 - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
}  // namespace

extern "C" int mma_lab(int kind, int ts, int n, int reps, long long* host) {
  long long* d;
  cudaMalloc(&d, 16);
  if (kind == 0 && !ts) k_mma<0, 0><<<1, 128>>>(n, reps, d);
  if (kind == 0 && ts) k_mma<0, 1><<<1, 128>>>(n, reps, d);
  if (kind == 1 && !ts) k_mma<1, 0><<<1, 128>>>(n, reps, d);
  if (kind == 1 && ts) k_mma<1, 1><<<1, 128>>>(n, reps, d);
  int e = (int)cudaDeviceSynchronize();
  cudaMemcpy(host, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}
