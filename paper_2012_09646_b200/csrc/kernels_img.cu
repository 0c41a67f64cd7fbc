// Image-processing (IMG) kernels for sm_100a (§V-B,
// Fig. 6; pipeline and constants: DESIGN.md reading R-IMG).
//
// The stencils (BLUR d=3/5, SOBEL 3x3) are HBM-bound (8 B/pixel of
// algorithmic traffic).  A direct 5x5 smem stencil would need 25 LDS per
// pixel and be shared-memory bound at ~1/3 of the HBM roofline, so both are
// computed SEPARABLY with a column-streaming scheme:
//   * a CTA owns 512 columns (128 threads x 4 columns) and a strip of rows;
//   * per input row it stages the row segment + halo in shared memory
//     (128-bit coalesced loads, double-buffered: one barrier per row),
//   * each thread applies the horizontal 1-D filter to its 4 columns from
//     smem (two 128-bit LDS), pushes the result into a register ring of the
//     last 2R+1 rows, and applies the vertical 1-D filter -> 4 outputs
//     stored with one 128-bit store.
// The normalised 2-D Gaussian exp(-(a^2+b^2)/2s^2)/Z equals the outer product
// of the normalised 1-D kernel, and Sobel Gx = [-1 0 1] (x) [1 2 1]^T,
// Gy = its transpose, so the results equal the 2-D definitions up to fp32
// rounding order.  Zero padding: out-of-range taps read 0.
#include "kcommon.cuh"

namespace dagrt {

constexpr int kImgThreads = 128;
constexpr int kImgCols = 4 * kImgThreads;  // 512 columns per CTA
constexpr int kImgRows = 64;               // default output rows per CTA (the host sizes grid.y)

// Horizontal/vertical 1-D filter functors.
template <int R>
struct GaussFilter {
  static constexpr int NCH = 1;
  float g[2 * R + 1];
  __device__ void init(float sigma2) {
    float s = 0.f;
#pragma unroll
    for (int k = -R; k <= R; ++k) {
      g[k + R] = expf(-(float)(k * k) / (2.0f * sigma2));
      s += g[k + R];
    }
#pragma unroll
    for (int k = 0; k < 2 * R + 1; ++k) g[k] /= s;
  }
  // win[j] = input at column c0 - R + j, j in [0, 4+2R)
  __device__ __forceinline__ void horiz(const float* win, float (&h)[NCH][4]) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float a = 0.f;
#pragma unroll
      for (int k = 0; k < 2 * R + 1; ++k) a = fmaf(g[k], win[q + k], a);
      h[0][q] = a;
    }
  }
  // ring[k] = horizontal result of row (y - R + k)
  __device__ __forceinline__ float vert(const float (&ring)[2 * R + 1][NCH][4], int q) const {
    float a = 0.f;
#pragma unroll
    for (int k = 0; k < 2 * R + 1; ++k) a = fmaf(g[k], ring[k][0][q], a);
    return a;
  }
};

struct SobelFilter {
  static constexpr int NCH = 2;  // channel 0: horizontal derivative, 1: horizontal smoothing
  __device__ void init(float) {}
  __device__ __forceinline__ void horiz(const float* win, float (&h)[NCH][4]) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h[0][q] = win[q + 2] - win[q];
      h[1][q] = win[q] + 2.0f * win[q + 1] + win[q + 2];
    }
  }
  __device__ __forceinline__ float vert(const float (&ring)[3][NCH][4], int q) const {
    const float gx = ring[0][0][q] + 2.0f * ring[1][0][q] + ring[2][0][q];
    const float gy = ring[2][1][q] - ring[0][1][q];
    return sqrtf(gx * gx + gy * gy);
  }
};

template <int R, typename F>
__device__ __forceinline__ void stencil_body(const float* __restrict__ src, float* __restrict__ dst,
                                             int H, int W, const F& f) {
  constexpr int D = 2 * R + 1;
  constexpr int ROWLEN = kImgCols + 2 * R + 4;  // + pad keeps both buffers 16-B aligned
  __shared__ __align__(16) float row[2][ROWLEN + (4 - (ROWLEN & 3)) % 4];
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * kImgCols;
  const int rows = (H + (int)gridDim.y - 1) / (int)gridDim.y;  // output rows per CTA (grid.y sets it)
  const int y0 = blockIdx.y * rows;
  const int y1 = min(H, y0 + rows);
  const int cx = x0 + 4 * t;  // first of this thread's 4 columns
  const bool vec = ((W & 3) == 0) && aligned16(src) && aligned16(dst);

  float ring[D][F::NCH][4];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int c = 0; c < F::NCH; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q) ring[k][c][q] = 0.f;

  // stage input row y (zero outside the image) into buffer b; smem index
  // j holds column x0 - R + j
  // Row staging is software-pipelined: the global loads of row y+1 (the
  // thread's 4 columns + halo) are issued before row y is filtered.
  struct RowRegs {
    float4 v;
    float h;  // halo element (threads t < R and t >= T-R)
  };
  auto load_row = [&](int y, RowRegs& rr) {
    rr.v = make_float4(0.f, 0.f, 0.f, 0.f);
    rr.h = 0.f;
    if (y >= 0 && y < H) {
      const float* s = src + (size_t)y * W;
      if (vec && cx + 3 < W) {
        rr.v = ldg_stream(reinterpret_cast<const float4*>(s + cx));
      } else {
        if (cx + 0 < W) rr.v.x = s[cx + 0];
        if (cx + 1 < W) rr.v.y = s[cx + 1];
        if (cx + 2 < W) rr.v.z = s[cx + 2];
        if (cx + 3 < W) rr.v.w = s[cx + 3];
      }
      if (t < R) {
        const int xl = x0 - R + t;
        rr.h = (xl >= 0) ? s[xl] : 0.f;
      } else if (t >= kImgThreads - R) {
        const int xr = x0 + kImgCols + (t - (kImgThreads - R));
        rr.h = (xr < W) ? s[xr] : 0.f;
      }
    }
  };
  auto store_row = [&](const RowRegs& rr, int b) {
    float* r = row[b];
    if (t < R) r[t] = rr.h;
    else if (t >= kImgThreads - R) r[R + kImgCols + (t - (kImgThreads - R))] = rr.h;
    r[R + 4 * t + 0] = rr.v.x;
    r[R + 4 * t + 1] = rr.v.y;
    r[R + 4 * t + 2] = rr.v.z;
    r[R + 4 * t + 3] = rr.v.w;
  };

  // prologue: rows y0-R .. y0+R-1 fill ring slots 1..D-1
  int b = 0;
  RowRegs cur;
  load_row(y0 - R, cur);
  for (int y = y0 - R; y < y1 + R; ++y, b ^= 1) {
    store_row(cur, b);
    if (y + 1 < y1 + R) load_row(y + 1, cur);
    __syncthreads();
    float win[4 + 2 * R];
#pragma unroll
    for (int j = 0; j < 4 + 2 * R; ++j) win[j] = row[b][4 * t + j];
    float h[F::NCH][4];
    f.horiz(win, h);
#pragma unroll
    for (int k = 0; k < D - 1; ++k)
#pragma unroll
      for (int c = 0; c < F::NCH; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) ring[k][c][q] = ring[k + 1][c][q];
#pragma unroll
    for (int c = 0; c < F::NCH; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q) ring[D - 1][c][q] = h[c][q];
    const int yo = y - R;  // output row completed by this input row
    if (yo >= y0 && cx < W) {
      float4 o;
      o.x = f.vert(ring, 0);
      o.y = f.vert(ring, 1);
      o.z = f.vert(ring, 2);
      o.w = f.vert(ring, 3);
      float* d = dst + (size_t)yo * W;
      if (vec && cx + 3 < W) {
        *reinterpret_cast<float4*>(d + cx) = o;
      } else {
        d[cx] = o.x;
        if (cx + 1 < W) d[cx + 1] = o.y;
        if (cx + 2 < W) d[cx + 2] = o.z;
        if (cx + 3 < W) d[cx + 3] = o.w;
      }
    }
    // the next iteration writes the other buffer; the barrier at its top
    // orders this iteration's reads of `row[b]` before the overwrite two
    // rows later
  }
}

// BLUR (Fig. 6): normalised Gaussian, diameter d in {3, 5}.
__global__ void __launch_bounds__(kImgThreads) k_blur(const float* __restrict__ src,
                                                      float* __restrict__ dst, int H, int W,
                                                      int diameter, float sigma2) {
  if (diameter == 3) {
    GaussFilter<1> f;
    f.init(sigma2);
    stencil_body<1>(src, dst, H, W, f);
  } else if (diameter == 5) {
    GaussFilter<2> f;
    f.init(sigma2);
    stencil_body<2>(src, dst, H, W, f);
  } else if (diameter == 1) {
    GaussFilter<0> f;
    f.init(sigma2);
    stencil_body<0>(src, dst, H, W, f);
  }
}

// SOBEL (Fig. 6): |grad| with the 3x3 Sobel taps.
__global__ void __launch_bounds__(kImgThreads) k_sobel(const float* __restrict__ src,
                                                       float* __restrict__ dst, int H, int W) {
  SobelFilter f;
  stencil_body<1>(src, dst, H, W, f);
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
