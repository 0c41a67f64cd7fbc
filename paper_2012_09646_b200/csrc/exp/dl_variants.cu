// Experimental DL variants (libdagrt_exp.so; see exp_common.cuh): conv1 with
// one output row per iteration, register caps for 1/3/4 CTAs per SM and
// evict-first stores, and the CUDA-core (FFMA) second convolution that the
// tcgen05 kernel replaced.  Same results as the product kernels.
#include "../conv1.cuh"
#include "exp_common.cuh"

namespace dagrt {

// the round-1/2 product conv1 (direct 64-byte-strided stores), for comparison
__global__ void __launch_bounds__(256, 3) k_conv1_r2b3(const float* __restrict__ x, const float* __restrict__ w,
                                                       float* __restrict__ out, int H, int W) {
  conv1_body2<false>(x, w, out, H, W);
}
__global__ void __launch_bounds__(256, 3) k_conv1_r2b3cs(const float* __restrict__ x, const float* __restrict__ w,
                                                         float* __restrict__ out, int H, int W) {
  conv1_body2<true>(x, w, out, H, W);
}
__global__ void __launch_bounds__(256, 2) k_conv1_r2b2(const float* __restrict__ x, const float* __restrict__ w,
                                                       float* __restrict__ out, int H, int W) {
  conv1_body2<false>(x, w, out, H, W);
}

// cp.async-staged, banded conv1 (conv1_body3): ring of 4 PFP + 5 input rows
// in dynamic shared memory (NSR x kConv1RowLen floats)
#define CONV1_CA(NAME, PFP, MINB, CS)                                                                  \
  __global__ void __launch_bounds__(256, MINB) NAME(const float* __restrict__ x, const float* __restrict__ w, \
                                                    float* __restrict__ out, int H, int W) {             \
    extern __shared__ __align__(16) float c1ring[];                                                    \
    conv1_body3<PFP, CS>(x, w, out, H, W, c1ring);                                                     \
  }
// conv1_body2 with warp-transposed (512-byte contiguous) stores
__global__ void __launch_bounds__(256, 3) k_conv1_r2b3st(const float* __restrict__ x, const float* __restrict__ w,
                                                         float* __restrict__ out, int H, int W) {
  conv1_body2<false, true>(x, w, out, H, W);
}
__global__ void __launch_bounds__(256, 3) k_conv1_r2b3stcs(const float* __restrict__ x, const float* __restrict__ w,
                                                           float* __restrict__ out, int H, int W) {
  conv1_body2<true, true>(x, w, out, H, W);
}
__global__ void __launch_bounds__(256, 4) k_conv1_r2b4st(const float* __restrict__ x, const float* __restrict__ w,
                                                         float* __restrict__ out, int H, int W) {
  conv1_body2<false, true>(x, w, out, H, W);
}
CONV1_CA(k_conv1_ca1b4, 1, 4, false)
CONV1_CA(k_conv1_ca1b3, 1, 3, false)
CONV1_CA(k_conv1_ca2b3, 2, 3, false)
CONV1_CA(k_conv1_ca2b4, 2, 4, false)
CONV1_CA(k_conv1_ca2b4cs, 2, 4, true)

__global__ void __launch_bounds__(256) k_conv1(const float* __restrict__ x, const float* __restrict__ w,
                                               float* __restrict__ out, int H, int W) {
  conv1_body(x, w, out, H, W);
}
// occupancy variants (same results): registers capped for 3 / 4 CTAs per SM
__global__ void __launch_bounds__(256, 3) k_conv1_b3(const float* __restrict__ x, const float* __restrict__ w,
                                                     float* __restrict__ out, int H, int W) {
  conv1_body(x, w, out, H, W);
}
__global__ void __launch_bounds__(256, 4) k_conv1_b4(const float* __restrict__ x, const float* __restrict__ w,
                                                     float* __restrict__ out, int H, int W) {
  conv1_body(x, w, out, H, W);
}
__global__ void __launch_bounds__(256, 4) k_conv1_b4cs(const float* __restrict__ x, const float* __restrict__ w,
                                                       float* __restrict__ out, int H, int W) {
  conv1_body<true>(x, w, out, H, W);
}

// CONV (second layer, 8 -> 16 channels).  One thread computes two
// horizontally adjacent output pixels (2-D grid, no integer division).  Per
// tap row it loads the 5 input pixels both outputs need (10 x LDG.128) and
// accumulates 2 x 16 outputs; the 16 x 72 weights sit in shared memory and
// are read with broadcast 128-bit loads, each reused for the two pixels.
__global__ void __launch_bounds__(256, 3) k_conv2(const float* __restrict__ in,
                                               const float* __restrict__ w,
                                               float* __restrict__ out, int H2, int W2) {
  __shared__ __align__(16) float sw[16 * 72];
  for (int i = threadIdx.x; i < 16 * 72; i += blockDim.x) sw[i] = w[i];
  __syncthreads();
  const int H3 = (H2 + 1) / 2, W3 = (W2 + 1) / 2;
  const int pairs = (W3 + 1) / 2;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= pairs) return;
  const float4* src = reinterpret_cast<const float4*>(in);
  for (int p = blockIdx.y; p < H3; p += gridDim.y) {
    float o[2][16];
#pragma unroll
    for (int k = 0; k < 16; ++k) { o[0][k] = 0.f; o[1][k] = 0.f; }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int y = 2 * p + a - 1;
      float4 v[5][2];  // input columns 4j-1 .. 4j+3
#pragma unroll
      for (int b = 0; b < 5; ++b) {
        const int xx = 4 * j - 1 + b;
        if (y >= 0 && y < H2 && xx >= 0 && xx < W2) {
          const size_t base = ((size_t)y * W2 + xx) * 2;
          v[b][0] = ldg_stream(src + base);
          v[b][1] = ldg_stream(src + base + 1);
        } else {
          v[b][0] = make_float4(0.f, 0.f, 0.f, 0.f);
          v[b][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const float4 w0 = *reinterpret_cast<const float4*>(sw + k * 72 + (a * 3 + b) * 8);
          const float4 w1 = *reinterpret_cast<const float4*>(sw + k * 72 + (a * 3 + b) * 8 + 4);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const float4 x0 = v[b + 2 * q][0], x1 = v[b + 2 * q][1];
            float s = o[q][k];
            s = fmaf(w0.x, x0.x, s);
            s = fmaf(w0.y, x0.y, s);
            s = fmaf(w0.z, x0.z, s);
            s = fmaf(w0.w, x0.w, s);
            s = fmaf(w1.x, x1.x, s);
            s = fmaf(w1.y, x1.y, s);
            s = fmaf(w1.z, x1.z, s);
            s = fmaf(w1.w, x1.w, s);
            o[q][k] = s;
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int qq = 2 * j + q;
      if (qq < W3) {
        float4* dst = reinterpret_cast<float4*>(out + ((size_t)p * W3 + qq) * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          dst[k] = make_float4(fmaxf(o[q][4 * k], 0.f), fmaxf(o[q][4 * k + 1], 0.f),
                               fmaxf(o[q][4 * k + 2], 0.f), fmaxf(o[q][4 * k + 3], 0.f));
      }
    }
  }
}

static const Builtin kDlExp[] = {
    {"conv1_r2b3st", (const void*)k_conv1_r2b3st, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_r2b3stcs", (const void*)k_conv1_r2b3stcs, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_r2b4st", (const void*)k_conv1_r2b4st, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_ca1b4", (const void*)k_conv1_ca1b4, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, 9 * 4112},
    {"conv1_ca1b3", (const void*)k_conv1_ca1b3, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, 9 * 4112},
    {"conv1_ca2b3", (const void*)k_conv1_ca2b3, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, 13 * 4112},
    {"conv1_ca2b4", (const void*)k_conv1_ca2b4, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, 13 * 4112},
    {"conv1_ca2b4cs", (const void*)k_conv1_ca2b4cs, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, 13 * 4112},
    {"conv1_b3", (const void*)k_conv1_b3, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_b4", (const void*)k_conv1_b4, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_b4cs", (const void*)k_conv1_b4cs, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_r2b3", (const void*)k_conv1_r2b3, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_r2b3cs", (const void*)k_conv1_r2b3cs, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_r2b2", (const void*)k_conv1_r2b2, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_b1", (const void*)k_conv1, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv2_ffma", (const void*)k_conv2, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
};
DAGRT_REGISTER_EXP(kDlExp);

}  // namespace dagrt
