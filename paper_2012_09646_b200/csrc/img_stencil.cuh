// Separable column-streaming stencil of the IMG kernels (kernels_img.cu,
// design notes there), shared with the experimental variants (exp/).
#pragma once
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

// PF = input rows whose global loads are in flight per thread (software
// pipeline depth of the row staging).
template <int R, typename F, int PF = 1>
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
  RowRegs pre[PF];
#pragma unroll
  for (int p = 0; p < PF; ++p) load_row(y0 - R + p < y1 + R ? y0 - R + p : -1, pre[p]);
  for (int y = y0 - R; y < y1 + R; ++y, b ^= 1) {
    store_row(pre[0], b);
#pragma unroll
    for (int p = 0; p + 1 < PF; ++p) pre[p] = pre[p + 1];
    if (y + PF < y1 + R) load_row(y + PF, pre[PF - 1]);
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

}  // namespace dagrt
