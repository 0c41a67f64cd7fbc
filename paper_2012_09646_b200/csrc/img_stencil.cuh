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


// The same stencil with the row staging done by cp.async (LDGSTS): every
// thread copies its 16 bytes (and the halo threads 4) of input row y + PF
// straight into a ring of PF + 1 shared-memory rows, so PF rows of loads are
// in flight per thread without holding them in registers (the register
// prefetch of stencil_body<PF > 1> cost occupancy).  Zero padding through the
// copies' source size (0 bytes read = 16 / 4 zero bytes written).  Row slot
// layout: index j holds column x0 - 4 + j (the 4-float left pad keeps every
// 16-byte destination aligned).  One CTA barrier per row, as before.
__device__ __forceinline__ void cp_async16(float* dst, const float* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

constexpr int kImgRowLen = kImgCols + 8;  // ring row: 4-float pads on both sides (R <= 4)
// ring_s: (PF + 1) x kImgRowLen floats of shared memory, 16-byte aligned (declared
// by the kernel, so that the instantiations for several R share it)
template <int R, typename F, int PF>
__device__ __forceinline__ void stencil_body_async(const float* __restrict__ src, float* __restrict__ dst,
                                                   int H, int W, const F& f, float (*ring_s)[kImgRowLen]) {
  constexpr int D = 2 * R + 1;
  constexpr int NS = PF + 1;            // ring slots
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * kImgCols;
  const int rows = (H + (int)gridDim.y - 1) / (int)gridDim.y;
  const int y0 = blockIdx.y * rows;
  const int y1 = min(H, y0 + rows);
  const int cx = x0 + 4 * t;
  const bool vec = ((W & 3) == 0) && aligned16(src) && aligned16(dst);

  float ring[D][F::NCH][4];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int c = 0; c < F::NCH; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q) ring[k][c][q] = 0.f;

  // issue the copies of input row y (zeros outside the image) into slot sl
  auto issue_row = [&](int y, int sl) {
    float* r = ring_s[sl];
    const bool in = y >= 0 && y < H;
    const float* s = src + (size_t)(in ? y : 0) * W;
    if (vec) {
      cp_async16(r + 4 + 4 * t, in && cx + 3 < W ? s + cx : src, in && cx + 3 < W ? 16 : 0);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        cp_async4(r + 4 + 4 * t + q, in && cx + q < W ? s + cx + q : src, in && cx + q < W ? 4 : 0);
    }
    if (t < R) {
      const int xl = x0 - R + t;
      cp_async4(r + 4 - R + t, in && xl >= 0 ? s + xl : src, in && xl >= 0 ? 4 : 0);
    } else if (t >= kImgThreads - R) {
      const int k = t - (kImgThreads - R);
      const int xr = x0 + kImgCols + k;
      cp_async4(r + 4 + kImgCols + k, in && xr < W ? s + xr : src, in && xr < W ? 4 : 0);
    }
  };

  const int ybeg = y0 - R, yend = y1 + R;  // input rows [ybeg, yend)
#pragma unroll
  for (int p = 0; p < PF; ++p) {
    if (ybeg + p < yend) issue_row(ybeg + p, p);
    cp_async_commit();  // one group per row (possibly empty): wait_group counts stay uniform
  }
  int sl = 0;
  for (int y = ybeg; y < yend; ++y) {
    cp_async_wait<PF - 1>();  // this thread's copies of row y have landed
    __syncthreads();          // ... everyone's; and everyone is done with row y - 1's slot
    const int ns = sl == 0 ? NS - 1 : sl - 1;  // slot of row y - 1 = slot of row y + PF
    if (y + PF < yend) issue_row(y + PF, ns);
    cp_async_commit();
    float win[4 + 2 * R];
#pragma unroll
    for (int j = 0; j < 4 + 2 * R; ++j) win[j] = ring_s[sl][4 - R + 4 * t + j];
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
    const int yo = y - R;
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
    sl = sl == NS - 1 ? 0 : sl + 1;
  }
  cp_async_wait<0>();
}

}  // namespace dagrt
