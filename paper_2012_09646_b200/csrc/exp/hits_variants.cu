// Experimental HITS L2-norm variant (tools/l2norm_lab.py): the vector streams
// through a per-CTA cp.async.bulk shared ring (NST chunks of CHB bytes in
// flight, one elected thread issues, an mbarrier per slot) instead of two
// 16-byte register loads per thread; the same fp32-per-float4 / fp64
// accumulation and deterministic grid finish as the product k_l2norm.
#include "../l2norm_ring.cuh"
#include "exp_common.cuh"

namespace dagrt {

#define L2N_TMA(NAME, NST, CHB, MINB)                                                                       \
  __global__ void __launch_bounds__(256, MINB) NAME(const float* __restrict__ v, RedOut* out, long long n) { \
    l2norm_tma_body<NST, CHB>(v, out, n);                                                                   \
  }
L2N_TMA(k_l2norm_t2x16, 2, 16384, 4)
L2N_TMA(k_l2norm_t3x12, 3, 12288, 4)
L2N_TMA(k_l2norm_t5x8, 5, 8192, 4)
L2N_TMA(k_l2norm_t4x8, 4, 8192, 6)

// the round-2 register form (two 16-byte streaming loads per thread in flight), for A/B
__global__ void __launch_bounds__(256, 8) k_l2norm_r2(const float* __restrict__ v, RedOut* out, long long n) {
  __shared__ double sh[32];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long long done = 0;
  if (aligned16(v)) {
    const long long n4 = n >> 2;
    const float4* v4 = reinterpret_cast<const float4*>(v);
    auto sq4 = [](float4 a) { return (double)fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, a.w * a.w))); };
    long long i = tid;
    for (; i + nth < n4; i += 2 * nth) {
      const float4 a = ldg_stream(v4 + i), b = ldg_stream(v4 + i + nth);
      acc += sq4(a) + sq4(b);
    }
    if (i < n4) acc += sq4(ldg_stream(v4 + i));
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) acc += (double)v[i] * v[i];
  double blk = block_reduce(acc, OpAdd(), sh);
  double total;
  if (grid_finish(out, blk, OpAdd(), 0.0, &total, sh) && threadIdx.x == 0) out->result = (float)sqrt(total);
}

static const Builtin kHitsExp2[] = {
    {"l2norm_r2", (const void*)k_l2norm_r2, "const ptr, out ptr, sint64", KF_NONE},
    {"l2norm_t2x16", (const void*)k_l2norm_t2x16, "const ptr, out ptr, sint64", KF_NONE},
    {"l2norm_t3x12", (const void*)k_l2norm_t3x12, "const ptr, out ptr, sint64", KF_NONE},
    {"l2norm_t5x8", (const void*)k_l2norm_t5x8, "const ptr, out ptr, sint64", KF_NONE},
    {"l2norm_t4x8", (const void*)k_l2norm_t4x8, "const ptr, out ptr, sint64", KF_NONE},
};
DAGRT_REGISTER_EXP(kHitsExp2);

}  // namespace dagrt
