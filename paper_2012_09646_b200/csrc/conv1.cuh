// First DL convolution (conv1: H x W x 1 -> H1 x W1 x 8, 3x3 stride 2
// pad 1, ReLU; §V-B, reading R-DL) -- the row bodies
// shared by the product kernel (kernels_dl.cu) and its occupancy / store
// policy variants (exp/dl_variants.cu).
#pragma once
#include "kcommon.cuh"

namespace dagrt {

// CONV (first layer): one thread computes two horizontally adjacent output
// pixels x 8 channels.  2-D grid: blockIdx.y walks output rows, x covers
// column pairs (no integer division).  Inputs: per tap row one float4
// (columns 4j..4j+3) plus column 4j-1 from the neighbouring lane (shuffle);
// outputs: 4 x 128-bit stores (64 contiguous bytes per thread).
// CS: stores with the evict-first (.cs) policy -- the 2 GB output streams
// through L2 without evicting the input rows the next output row re-reads.
template <bool CS = false>
__device__ __forceinline__ void conv1_body(const float* __restrict__ x, const float* __restrict__ w,
                                           float* __restrict__ out, int H, int W) {
  const int H1 = (H + 1) / 2, W1 = (W + 1) / 2;
  const int pairs = (W1 + 1) / 2;
  // weights in shared memory (uniform 128-bit broadcast reads): keeping all
  // 72 in registers would cap occupancy at 25% and starve the loads
  __shared__ __align__(16) float wr[72];
  if (threadIdx.x < 72) wr[threadIdx.x] = __ldg(w + threadIdx.x);
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live_j = j < pairs;
  const bool vec = ((W & 3) == 0) && aligned16(x);
  const int c0 = 4 * j;
  // the three input rows of output row p (one float4 each); the next row's
  // loads are issued before this row is computed (software pipelining)
  auto load_rows = [&](int p, float4 (&q)[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int y = 2 * p + a - 1;
      q[a] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (live_j && y >= 0 && y < H) {
        const float* row = x + (size_t)y * W;
        if (vec && c0 + 3 < W) {
          q[a] = ldg_stream(reinterpret_cast<const float4*>(row + c0));
        } else {
          if (c0 + 0 < W) q[a].x = row[c0 + 0];
          if (c0 + 1 < W) q[a].y = row[c0 + 1];
          if (c0 + 2 < W) q[a].z = row[c0 + 2];
          if (c0 + 3 < W) q[a].w = row[c0 + 3];
        }
      }
    }
  };
  float4 q[3];
  if ((int)blockIdx.y < H1) load_rows(blockIdx.y, q);
  for (int p = blockIdx.y; p < H1; p += gridDim.y) {  // uniform per block
    float4 qn[3];
    if (p + (int)gridDim.y < H1) load_rows(p + gridDim.y, qn);
    float v[3][5];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int y = 2 * p + a - 1;
      const bool rowok = live_j && y >= 0 && y < H;
      float left = __shfl_up_sync(0xffffffffu, q[a].w, 1);
      if ((threadIdx.x & 31) == 0 || j == 0) left = (rowok && c0 > 0) ? x[(size_t)y * W + c0 - 1] : 0.f;
      v[a][0] = left;
      v[a][1] = q[a].x;
      v[a][2] = q[a].y;
      v[a][3] = q[a].z;
      v[a][4] = q[a].w;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) q[a] = qn[a];
    if (!live_j) continue;
    float o[2][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const float ww = wr[k * 9 + a * 3 + b];
          s0 = fmaf(ww, v[a][b], s0);      // q = 2j   -> cols 4j-1+b
          s1 = fmaf(ww, v[a][b + 2], s1);  // q = 2j+1 -> cols 4j+1+b
        }
      o[0][k] = fmaxf(s0, 0.f);
      o[1][k] = fmaxf(s1, 0.f);
    }
    float4* dst = reinterpret_cast<float4*>(out + ((size_t)p * W1 + 2 * j) * 8);
    auto st = [&](float4* d, float4 v) {
      if (CS) __stcs(d, v);
      else *d = v;
    };
    st(dst + 0, make_float4(o[0][0], o[0][1], o[0][2], o[0][3]));
    st(dst + 1, make_float4(o[0][4], o[0][5], o[0][6], o[0][7]));
    if (2 * j + 1 < W1) {
      st(dst + 2, make_float4(o[1][0], o[1][1], o[1][2], o[1][3]));
      st(dst + 3, make_float4(o[1][4], o[1][5], o[1][6], o[1][7]));
    }
  }
}

// Two output rows per iteration: rows 2r and 2r+1 share input row 4r+1, so
// 5 input rows are loaded per 2 output rows (6 for two single-row
// iterations) and each thread has twice the independent loads and stores in
// flight; the next pair's 5 rows are loaded before this pair is computed.
template <bool CS>
__device__ __forceinline__ void conv1_body2(const float* __restrict__ x, const float* __restrict__ w,
                                            float* __restrict__ out, int H, int W) {
  const int H1 = (H + 1) / 2, W1 = (W + 1) / 2;
  const int pairs = (W1 + 1) / 2;
  __shared__ __align__(16) float wr[72];
  if (threadIdx.x < 72) wr[threadIdx.x] = __ldg(w + threadIdx.x);
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live_j = j < pairs;
  const bool vec = ((W & 3) == 0) && aligned16(x);
  const int c0 = 4 * j;
  const int R = (H1 + 1) / 2;  // output row pairs
  auto load_rows = [&](int r, float4 (&q)[5]) {
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int y = 4 * r + a - 1;
      q[a] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (live_j && y >= 0 && y < H) {
        const float* row = x + (size_t)y * W;
        if (vec && c0 + 3 < W) {
          q[a] = ldg_stream(reinterpret_cast<const float4*>(row + c0));
        } else {
          if (c0 + 0 < W) q[a].x = row[c0 + 0];
          if (c0 + 1 < W) q[a].y = row[c0 + 1];
          if (c0 + 2 < W) q[a].z = row[c0 + 2];
          if (c0 + 3 < W) q[a].w = row[c0 + 3];
        }
      }
    }
  };
  float4 q[5];
  if ((int)blockIdx.y < R) load_rows(blockIdx.y, q);
  for (int r = blockIdx.y; r < R; r += gridDim.y) {  // uniform per block
    float4 qn[5];
    if (r + (int)gridDim.y < R) load_rows(r + gridDim.y, qn);
    float v[5][5];
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int y = 4 * r + a - 1;
      const bool rowok = live_j && y >= 0 && y < H;
      float left = __shfl_up_sync(0xffffffffu, q[a].w, 1);
      if ((threadIdx.x & 31) == 0 || j == 0) left = (rowok && c0 > 0) ? x[(size_t)y * W + c0 - 1] : 0.f;
      v[a][0] = left;
      v[a][1] = q[a].x;
      v[a][2] = q[a].y;
      v[a][3] = q[a].z;
      v[a][4] = q[a].w;
    }
#pragma unroll
    for (int a = 0; a < 5; ++a) q[a] = qn[a];
    if (!live_j) continue;
    // output row p = 2r + h from input rows v[2h .. 2h+2]; the memory clobber
    // between the two rows keeps the compiler from holding all 72 weights in
    // registers across them (it re-reads the broadcast smem copy instead)
    auto row = [&](int h, const float (&v0)[5], const float (&v1)[5], const float (&v2)[5]) {
      const int p = 2 * r + h;
      if (p >= H1) return;
      const float* vr[3] = {v0, v1, v2};
      float o[2][8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const float ww = wr[k * 9 + a * 3 + b];
            s0 = fmaf(ww, vr[a][b], s0);
            s1 = fmaf(ww, vr[a][b + 2], s1);
          }
        o[0][k] = fmaxf(s0, 0.f);
        o[1][k] = fmaxf(s1, 0.f);
      }
      float4* dst = reinterpret_cast<float4*>(out + ((size_t)p * W1 + 2 * j) * 8);
      auto st = [&](float4* d, float4 val) {
        if (CS) __stcs(d, val);
        else *d = val;
      };
      st(dst + 0, make_float4(o[0][0], o[0][1], o[0][2], o[0][3]));
      st(dst + 1, make_float4(o[0][4], o[0][5], o[0][6], o[0][7]));
      if (2 * j + 1 < W1) {
        st(dst + 2, make_float4(o[1][0], o[1][1], o[1][2], o[1][3]));
        st(dst + 3, make_float4(o[1][4], o[1][5], o[1][6], o[1][7]));
      }
    };
    row(0, v[0], v[1], v[2]);
    asm volatile("" ::: "memory");
    row(1, v[2], v[3], v[4]);
  }
}

}  // namespace dagrt
