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

static const Builtin kHitsExp2[] = {
    {"l2norm_t2x16", (const void*)k_l2norm_t2x16, "const ptr, out ptr, sint64", KF_NONE},
    {"l2norm_t3x12", (const void*)k_l2norm_t3x12, "const ptr, out ptr, sint64", KF_NONE},
    {"l2norm_t5x8", (const void*)k_l2norm_t5x8, "const ptr, out ptr, sint64", KF_NONE},
    {"l2norm_t4x8", (const void*)k_l2norm_t4x8, "const ptr, out ptr, sint64", KF_NONE},
};
DAGRT_REGISTER_EXP(kHitsExp2);

}  // namespace dagrt
