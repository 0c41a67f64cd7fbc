// HITS L2 norm through a per-CTA cp.async.bulk shared ring (the product
// "l2norm", kernels_hits.cu, and its experimental shapes, exp/hits_variants.cu):
// each CTA of a persistent grid streams a contiguous range of the vector in
// chunks of CHB bytes, NST in flight (one elected thread issues, an mbarrier
// per slot), squares summed in fp32 per float4 and accumulated in fp64, the
// grid finished deterministically (RedOut).  ncu on the round-2 register
// form (two 16-byte loads per thread in flight): long-scoreboard stalls
// dominated, 19.4 us per 20M floats; tools/l2norm_lab.py.
#pragma once
#include "kcommon.cuh"

namespace dagrt {

__device__ __forceinline__ void hv_mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)));
}
__device__ __forceinline__ void hv_mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void hv_bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"(b) : "memory");
}

template <int NST, int CHB>
__device__ __forceinline__ void l2norm_tma_body(const float* __restrict__ v, RedOut* out, long long n) {
  constexpr int CF4 = CHB / 16;  // float4 per chunk
  __shared__ __align__(128) float4 ring[NST][CF4];
  __shared__ uint64_t full[NST];
  __shared__ double sh[32];
  const int t = threadIdx.x;
  auto sq4 = [](float4 a) { return (double)fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, a.w * a.w))); };
  double acc = 0.0;
  const long long G = gridDim.x;
  const long long n4 = aligned16(v) ? n >> 2 : 0;
  // contiguous range of float4 per CTA, whole chunks through the ring
  const long long per = (n4 + G - 1) / G;
  const long long b0 = min(n4, (long long)blockIdx.x * per), b1 = min(n4, b0 + per);
  const long long nch = (b1 - b0) / CF4;
  const float4* v4 = reinterpret_cast<const float4*>(v);
  if (t == 0) {
    for (int s = 0; s < NST; ++s) hv_mbar_init(&full[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NST && s < nch; ++s) hv_bulk(ring[s], v4 + b0 + (long long)s * CF4, CHB, &full[s]);
  }
  __syncthreads();
  for (long long c = 0; c < nch; ++c) {
    const int st = (int)(c % NST);
    hv_mbar_wait(&full[st], (unsigned)((c / NST) & 1));
    double a = 0.0;
#pragma unroll
    for (int k = t; k < CF4; k += blockDim.x) a += sq4(ring[st][k]);
    acc += a;
    __syncthreads();
    if (t == 0 && c + NST < nch) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      hv_bulk(ring[st], v4 + b0 + (c + NST) * CF4, CHB, &full[st]);
    }
  }
  for (long long i = b0 + nch * CF4 + t; i < b1; i += blockDim.x) acc += sq4(__ldg(v4 + i));
  for (long long i = (n4 << 2) + (long long)blockIdx.x * blockDim.x + t; i < n; i += G * blockDim.x)
    acc += (double)v[i] * v[i];
  double blk = block_reduce(acc, OpAdd(), sh);
  double total;
  if (grid_finish(out, blk, OpAdd(), 0.0, &total, sh) && threadIdx.x == 0) out->result = (float)sqrt(total);
}

}  // namespace dagrt
