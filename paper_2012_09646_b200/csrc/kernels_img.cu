// Image-processing (IMG) kernels for sm_100a (§V-B,
// Fig. 6; pipeline and constants: DESIGN.md reading R-IMG).
//
// The stencils (BLUR d=3/5, SOBEL 3x3) are HBM-bound (8 B/pixel of
// algorithmic traffic).  A direct 5x5 smem stencil would need 25 LDS per
// pixel and be shared-memory bound at ~1/3 of the HBM roofline, so both are
// computed SEPARABLY with a column-streaming scheme:
//   * a CTA owns 512 columns (128 threads x 4 columns) and a strip of rows;
//   * per input row it stages the row segment + halo in shared memory with
//     cp.async (16-byte copies, zero-filled outside the image) into a ring
//     of PF + 1 rows, PF rows ahead (one barrier per row),
//   * each thread applies the horizontal 1-D filter to its 4 columns from
//     smem (two 128-bit LDS), pushes the result into a register ring of the
//     last 2R+1 rows, and applies the vertical 1-D filter -> 4 outputs
//     stored with one 128-bit store.
// The normalised 2-D Gaussian exp(-(a^2+b^2)/2s^2)/Z equals the outer product
// of the normalised 1-D kernel, and Sobel Gx = [-1 0 1] (x) [1 2 1]^T,
// Gy = its transpose, so the results equal the 2-D definitions up to fp32
// rounding order.  Zero padding: out-of-range taps read 0.
#include "img_stencil.cuh"

namespace dagrt {

// BLUR (Fig. 6): normalised Gaussian, diameter d in {3, 5}.
// Row staging by cp.async into a ring of kBlurPF + 1 rows (img_stencil.cuh
// stencil_body_async): 358 vs 431 us per 16384^2 launch with the round-1
// register-staged rows (0.92 vs 0.76 of HBM, bitwise-identical outputs,
// tools/img_variants.py, profiles/r2_img_stencil_variants.json).
constexpr int kBlurPF = 4, kSobelPF = 6;
__global__ void __launch_bounds__(kImgThreads) k_blur(const float* __restrict__ src,
                                                      float* __restrict__ dst, int H, int W,
                                                      int diameter, float sigma2) {
  __shared__ __align__(16) float ring_s[kBlurPF + 1][kImgRowLen];
  if (diameter == 3) {
    GaussFilter<1> f;
    f.init(sigma2);
    stencil_body_async<1, GaussFilter<1>, kBlurPF>(src, dst, H, W, f, ring_s);
  } else if (diameter == 5) {
    GaussFilter<2> f;
    f.init(sigma2);
    stencil_body_async<2, GaussFilter<2>, kBlurPF>(src, dst, H, W, f, ring_s);
  } else if (diameter == 1) {
    GaussFilter<0> f;
    f.init(sigma2);
    stencil_body_async<0, GaussFilter<0>, kBlurPF>(src, dst, H, W, f, ring_s);
  }
}

// SOBEL (Fig. 6): |grad| with the 3x3 Sobel taps (367 vs 453 us, 0.90 of HBM).
__global__ void __launch_bounds__(kImgThreads) k_sobel(const float* __restrict__ src,
                                                       float* __restrict__ dst, int H, int W) {
  __shared__ __align__(16) float ring_s[kSobelPF + 1][kImgRowLen];
  SobelFilter f;
  stencil_body_async<1, SobelFilter, kSobelPF>(src, dst, H, W, f, ring_s);
}

// MAX / MIN (Fig. 6): global extrema of the sobel mask (two sibling
// vertices on different streams).
template <bool IS_MAX>
__global__ void __launch_bounds__(256) k_extremum(const float* __restrict__ x, RedOut* out,
                                                  long long n) {
  __shared__ double sh[32];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  float acc = IS_MAX ? -INFINITY : INFINITY;
  long long done = 0;
  if (aligned16(x)) {
    const long long n4 = n >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    long long i = tid;
    for (; i + nth < n4; i += 2 * nth) {
      float4 a = ldg_stream(x4 + i), b = ldg_stream(x4 + i + nth);
      if (IS_MAX) acc = fmaxf(acc, fmaxf(fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)),
                                         fmaxf(fmaxf(b.x, b.y), fmaxf(b.z, b.w))));
      else acc = fminf(acc, fminf(fminf(fminf(a.x, a.y), fminf(a.z, a.w)),
                                  fminf(fminf(b.x, b.y), fminf(b.z, b.w))));
    }
    for (; i < n4; i += nth) {
      float4 a = ldg_stream(x4 + i);
      if (IS_MAX) acc = fmaxf(acc, fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)));
      else acc = fminf(acc, fminf(fminf(a.x, a.y), fminf(a.z, a.w)));
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) acc = IS_MAX ? fmaxf(acc, x[i]) : fminf(acc, x[i]);
  double v = (double)acc;
  double blk = IS_MAX ? block_reduce(v, OpMax(), sh) : block_reduce(v, OpMin(), sh);
  double total;
  bool last = IS_MAX ? grid_finish(out, blk, OpMax(), -INFINITY, &total, sh)
                     : grid_finish(out, blk, OpMin(), INFINITY, &total, sh);
  if (last && threadIdx.x == 0) out->result = (float)total;
}

// EXTEND (Fig. 6), in place: m = min(1, factor (m - mn)/(mx - mn)); 0 if mx == mn.
__global__ void __launch_bounds__(256) k_extend(float* __restrict__ m, const RedOut* __restrict__ mx,
                                                const RedOut* __restrict__ mn, long long n,
                                                float factor) {
  const float hi = mx->result, lo = mn->result;
  const float scale = (hi > lo) ? factor / (hi - lo) : 0.f;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(m)) {
    const long long n4 = n >> 2;
    float4* m4 = reinterpret_cast<float4*>(m);
    for (long long i = tid; i < n4; i += nth) {
      float4 v = m4[i];
      v.x = fminf(1.f, (v.x - lo) * scale);
      v.y = fminf(1.f, (v.y - lo) * scale);
      v.z = fminf(1.f, (v.z - lo) * scale);
      v.w = fminf(1.f, (v.w - lo) * scale);
      m4[i] = v;
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) m[i] = fminf(1.f, (m[i] - lo) * scale);
}

// UNSHARPEN (Fig. 6): clamp(x (1+a) - blur a, 0, 1).
__global__ void __launch_bounds__(256) k_unsharpen(const float* __restrict__ x,
                                                   const float* __restrict__ bl,
                                                   float* __restrict__ out, long long n,
                                                   float amount) {
  const float a1 = 1.f + amount;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(x) && aligned16(bl) && aligned16(out)) {
    const long long n4 = n >> 2;
    for (long long i = tid; i < n4; i += nth) {
      float4 u = ldg_stream(reinterpret_cast<const float4*>(x) + i);
      float4 b = ldg_stream(reinterpret_cast<const float4*>(bl) + i);
      float4 o;
      o.x = __saturatef(u.x * a1 - b.x * amount);
      o.y = __saturatef(u.y * a1 - b.y * amount);
      o.z = __saturatef(u.z * a1 - b.z * amount);
      o.w = __saturatef(u.w * a1 - b.w * amount);
      reinterpret_cast<float4*>(out)[i] = o;
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) out[i] = __saturatef(x[i] * a1 - bl[i] * amount);
}

// COMBINE (Fig. 6): x m + y (1 - m).
__global__ void __launch_bounds__(256) k_combine(const float* __restrict__ x,
                                                 const float* __restrict__ y,
                                                 const float* __restrict__ m,
                                                 float* __restrict__ out, long long n) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(x) && aligned16(y) && aligned16(m) && aligned16(out)) {
    const long long n4 = n >> 2;
    for (long long i = tid; i < n4; i += nth) {
      float4 a = ldg_stream(reinterpret_cast<const float4*>(x) + i);
      float4 b = ldg_stream(reinterpret_cast<const float4*>(y) + i);
      float4 w = ldg_stream(reinterpret_cast<const float4*>(m) + i);
      float4 o;
      o.x = a.x * w.x + b.x * (1.f - w.x);
      o.y = a.y * w.y + b.y * (1.f - w.y);
      o.z = a.z * w.z + b.z * (1.f - w.z);
      o.w = a.w * w.w + b.w * (1.f - w.w);
      reinterpret_cast<float4*>(out)[i] = o;
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) out[i] = x[i] * m[i] + y[i] * (1.f - m[i]);
}

// launch contracts (dagrt_launch validates them; builtin.h LaunchCheck)
static const char* v_stencil(const LaunchCheck& L) {  // src, dst, H, W [, d, sigma^2]
  const uint64_t n = (uint64_t)(uint32_t)L.i32(2) * (uint32_t)L.i32(3);
  if (L.i32(2) < 0 || L.i32(3) < 0) return "negative image size";
  if (!fits(L, 0, 4 * n) || !fits(L, 1, 4 * n)) return "images need 4 H W bytes";
  if (L.block[0] != 128 || L.block[1] != 1 || L.block[2] != 1) return "the stencil tile needs 128 threads";
  if (L.nargs > 4 && L.i32(4) != 1 && L.i32(4) != 3 && L.i32(4) != 5) return "blur diameter must be 1, 3 or 5";
  return nullptr;
}
static const char* v_extremum(const LaunchCheck& L) {
  if (!fits(L, 0, 4 * (uint64_t)L.i(2))) return "input needs 4 n bytes";
  return check_reduction(L, 1);
}
static const char* v_extend(const LaunchCheck& L) {
  if (!fits(L, 0, 4 * (uint64_t)L.i(3))) return "mask needs 4 n bytes";
  return fits(L, 1, 4) && fits(L, 2, 4) ? nullptr : "extrema outputs too small";
}
template <int NA>  // NA fp32 arrays of n elements, then n
static const char* v_pointwise(const LaunchCheck& L) {
  const uint64_t n = (uint64_t)L.i(NA);
  for (int a = 0; a < NA; ++a)
    if (!fits(L, a, 4 * n)) return "arrays need 4 n bytes";
  return nullptr;
}

static const Builtin kImg[] = {
    {"blur", (const void*)k_blur, "const ptr, out ptr, sint32, sint32, sint32, float", KF_NONE, 0, nullptr, v_stencil},
    {"sobel", (const void*)k_sobel, "const ptr, out ptr, sint32, sint32", KF_NONE, 0, nullptr, v_stencil},
    {"maximum", (const void*)k_extremum<true>, "const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_extremum},
    {"minimum", (const void*)k_extremum<false>, "const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_extremum},
    {"extend", (const void*)k_extend, "ptr, const ptr, const ptr, sint64, float", KF_NONE, 0, nullptr, v_extend},
    {"unsharpen", (const void*)k_unsharpen, "const ptr, const ptr, out ptr, sint64, float", KF_NONE, 0, nullptr, v_pointwise<3>},
    {"combine", (const void*)k_combine, "const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_pointwise<4>},
};
DAGRT_REGISTER_BUILTINS(kImg);

}  // namespace dagrt
