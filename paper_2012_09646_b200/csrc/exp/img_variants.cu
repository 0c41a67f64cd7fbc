// Experimental IMG stencil variants (tools/img_variants.py): the product
// column-streaming stencil (img_stencil.cuh) with PF input rows of global
// loads in flight per thread instead of one.  ncu on the product k_blur
// (profiles/r2_summary.md): long-scoreboard and barrier stalls lead, 0.77 of
// HBM -- one 16-byte load per thread in flight is too little for HBM latency.
#include "../img_stencil.cuh"
#include "exp_common.cuh"

namespace dagrt {

template <int PF>
__device__ __forceinline__ void blur_pf(const float* __restrict__ src, float* __restrict__ dst, int H, int W,
                                        int diameter, float sigma2) {
  if (diameter == 3) {
    GaussFilter<1> f;
    f.init(sigma2);
    stencil_body<1, GaussFilter<1>, PF>(src, dst, H, W, f);
  } else if (diameter == 5) {
    GaussFilter<2> f;
    f.init(sigma2);
    stencil_body<2, GaussFilter<2>, PF>(src, dst, H, W, f);
  } else if (diameter == 1) {
    GaussFilter<0> f;
    f.init(sigma2);
    stencil_body<0, GaussFilter<0>, PF>(src, dst, H, W, f);
  }
}
#define IMG_PF_VARIANTS(PF)                                                                          \
  __global__ void __launch_bounds__(kImgThreads) k_blur_pf##PF(const float* __restrict__ src,        \
                                                               float* __restrict__ dst, int H, int W, \
                                                               int diameter, float sigma2) {         \
    blur_pf<PF>(src, dst, H, W, diameter, sigma2);                                                   \
  }                                                                                                  \
  __global__ void __launch_bounds__(kImgThreads) k_sobel_pf##PF(const float* __restrict__ src,       \
                                                                float* __restrict__ dst, int H, int W) { \
    SobelFilter f;                                                                                   \
    stencil_body<1, SobelFilter, PF>(src, dst, H, W, f);                                             \
  }
IMG_PF_VARIANTS(1)
IMG_PF_VARIANTS(2)
IMG_PF_VARIANTS(3)
IMG_PF_VARIANTS(4)

template <int PF>
__device__ __forceinline__ void blur_ca(const float* __restrict__ src, float* __restrict__ dst, int H, int W,
                                        int diameter, float sigma2) {
  __shared__ __align__(16) float ring_s[PF + 1][kImgRowLen];
  if (diameter == 3) {
    GaussFilter<1> f;
    f.init(sigma2);
    stencil_body_async<1, GaussFilter<1>, PF>(src, dst, H, W, f, ring_s);
  } else if (diameter == 5) {
    GaussFilter<2> f;
    f.init(sigma2);
    stencil_body_async<2, GaussFilter<2>, PF>(src, dst, H, W, f, ring_s);
  } else if (diameter == 1) {
    GaussFilter<0> f;
    f.init(sigma2);
    stencil_body_async<0, GaussFilter<0>, PF>(src, dst, H, W, f, ring_s);
  }
}
#define IMG_CA_VARIANTS(PF)                                                                          \
  __global__ void __launch_bounds__(kImgThreads) k_blur_ca##PF(const float* __restrict__ src,        \
                                                               float* __restrict__ dst, int H, int W, \
                                                               int diameter, float sigma2) {         \
    blur_ca<PF>(src, dst, H, W, diameter, sigma2);                                                   \
  }                                                                                                  \
  __global__ void __launch_bounds__(kImgThreads) k_sobel_ca##PF(const float* __restrict__ src,       \
                                                                float* __restrict__ dst, int H, int W) { \
    __shared__ __align__(16) float ring_s[PF + 1][kImgRowLen];                                       \
    SobelFilter f;                                                                                   \
    stencil_body_async<1, SobelFilter, PF>(src, dst, H, W, f, ring_s);                               \
  }
IMG_CA_VARIANTS(2)
IMG_CA_VARIANTS(3)
IMG_CA_VARIANTS(4)
IMG_CA_VARIANTS(6)

static const Builtin kImgExp[] = {
#define IMG_PF_REG(PF)                                                                                           \
  {"blur_pf" #PF, (const void*)k_blur_pf##PF, "const ptr, out ptr, sint32, sint32, sint32, float", KF_NONE}, \
      {"sobel_pf" #PF, (const void*)k_sobel_pf##PF, "const ptr, out ptr, sint32, sint32", KF_NONE},
    IMG_PF_REG(1) IMG_PF_REG(2) IMG_PF_REG(3) IMG_PF_REG(4)
#define IMG_CA_REG(PF)                                                                                           \
  {"blur_ca" #PF, (const void*)k_blur_ca##PF, "const ptr, out ptr, sint32, sint32, sint32, float", KF_NONE}, \
      {"sobel_ca" #PF, (const void*)k_sobel_ca##PF, "const ptr, out ptr, sint32, sint32", KF_NONE},
    IMG_CA_REG(2) IMG_CA_REG(3) IMG_CA_REG(4) IMG_CA_REG(6)
};
DAGRT_REGISTER_EXP(kImgExp);

}  // namespace dagrt
