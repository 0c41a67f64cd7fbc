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
// ST (staged stores): each warp transposes its 2 KB of outputs per row
// through shared memory (swizzled: conflict-free both ways) so that every
// 128-bit store instruction covers 512 contiguous bytes (4 lines) instead of
// 16 B at a 64 B stride (16 lines, half sectors).
template <bool CS, bool ST = false>
__device__ __forceinline__ void conv1_body2(const float* __restrict__ x, const float* __restrict__ w,
                                            float* __restrict__ out, int H, int W) {
  const int H1 = (H + 1) / 2, W1 = (W + 1) / 2;
  const int pairs = (W1 + 1) / 2;
  __shared__ __align__(16) float4 stg[ST ? 8 : 1][32][4];  // [warp][lane][slot]
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
    if (!ST && !live_j) continue;  // (ST: the whole warp takes part in the staged stores)
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
      auto st = [&](float4* d, float4 val) {
        if (CS) __stcs(d, val);
        else *d = val;
      };
      if (ST) {
        const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
        float4(*sm)[4] = stg[ST ? wp : 0];
        const int sw = (lane >> 1) & 3;
        __syncwarp();  // the previous row's reads of this warp's slots are done
        sm[lane][0 ^ sw] = make_float4(o[0][0], o[0][1], o[0][2], o[0][3]);
        sm[lane][1 ^ sw] = make_float4(o[0][4], o[0][5], o[0][6], o[0][7]);
        sm[lane][2 ^ sw] = make_float4(o[1][0], o[1][1], o[1][2], o[1][3]);
        sm[lane][3 ^ sw] = make_float4(o[1][4], o[1][5], o[1][6], o[1][7]);
        __syncwarp();
        const int j0 = j - lane;  // column pair of lane 0
        float4* dst0 = reinterpret_cast<float4*>(out + ((size_t)p * W1 + 2 * j0) * 8);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int e = 32 * k + lane;           // float4 of the warp's 2 KB
          const int ow = e >> 2, qq = e & 3;     // owner lane, its slot
          const int jo = j0 + ow;
          const float4 val = sm[ow][qq ^ ((ow >> 1) & 3)];
          if (jo < pairs && (qq < 2 || 2 * jo + 1 < W1)) st(dst0 + e, val);
        }
        return;
      }
      float4* dst = reinterpret_cast<float4*>(out + ((size_t)p * W1 + 2 * j) * 8);
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


// Two output rows per iteration with the input rows staged by cp.async
// (LDGSTS) into a shared-memory ring, PFP row pairs ahead, and each CTA
// walking a contiguous BAND of row pairs (blockIdx.y) so that the input row
// shared by consecutive pairs (4r + 3) is copied once: 4 new rows per pair.
// No prefetch registers (the register-pipelined conv1_body2 held 5 float4 in
// flight at 80 registers, 3 CTAs/SM: long-scoreboard stalls led, ncu).  A CTA
// covers 1024 input columns (256 threads x 4); ring row index 4 + 4t holds
// column x0 + 4t, index 3 column x0 - 1 (zero at the image border).  The
// arithmetic and its order are conv1_body2's: bitwise-identical outputs.
constexpr int kConv1RowLen = 4 + 1024;  // floats per ring row (16-byte multiple)
__device__ __forceinline__ void c1_cp16(float* dst, const float* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void c1_cp4(float* dst, const float* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes) : "memory");
}
template <int PFP, bool CS>
__device__ __forceinline__ void conv1_body3(const float* __restrict__ x, const float* __restrict__ w,
                                            float* __restrict__ out, int H, int W, float* ring /* NSR x kConv1RowLen */) {
  constexpr int NSR = 4 * PFP + 5;  // ring rows: pair k's 5 rows + PFP pairs of 4 ahead
  const int H1 = (H + 1) / 2, W1 = (W + 1) / 2;
  const int pairs = (W1 + 1) / 2;
  __shared__ __align__(16) float wr[72];
  if (threadIdx.x < 72) wr[threadIdx.x] = __ldg(w + threadIdx.x);
  const int t = threadIdx.x;
  const int j = blockIdx.x * blockDim.x + t;
  const bool live_j = j < pairs;
  const int x0 = blockIdx.x * 4 * (int)blockDim.x;
  const int c0 = 4 * j;
  const bool vec = ((W & 3) == 0) && aligned16(x);
  const int RP = (H1 + 1) / 2;  // output row pairs
  const int per = (RP + (int)gridDim.y - 1) / (int)gridDim.y;
  const int rb = blockIdx.y * per, re = min(RP, rb + per);
  if (rb >= re) return;  // uniform per block (before any barrier)
  const int ybase = 4 * rb - 1;           // input row of ring index i: ybase + i
  const int ilast = 4 * (re - rb);        // last input row index the band needs
  auto issue = [&](int i) {               // copies of input row index i into slot i % NSR
    float* r = ring + (size_t)(i % NSR) * kConv1RowLen;
    const int y = ybase + i;
    const bool in = y >= 0 && y < H;
    const float* row = x + (size_t)(in ? y : 0) * W;
    if (vec) {
      const bool ok = in && live_j && c0 + 3 < W;
      c1_cp16(r + 4 + 4 * t, ok ? row + c0 : x, ok ? 16 : 0);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool ok = in && live_j && c0 + q < W;
        c1_cp4(r + 4 + 4 * t + q, ok ? row + c0 + q : x, ok ? 4 : 0);
      }
    }
    if (t == 0) {
      const bool ok = in && x0 > 0;
      c1_cp4(r + 3, ok ? row + x0 - 1 : x, ok ? 4 : 0);
    }
  };
  // group 0: rows 0..4 (pair 0); group p: rows 4p+1 .. 4p+4
#pragma unroll
  for (int p = 0; p < PFP; ++p) {
    for (int i = (p == 0 ? 0 : 4 * p + 1); i <= 4 * p + 4; ++i)
      if (i <= ilast) issue(i);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int k = 0; rb + k < re; ++k) {
    asm volatile("cp.async.wait_group %0;" ::"n"(PFP - 1) : "memory");
    __syncthreads();  // pair k's rows landed for every thread; pair k-1's slots are free
    {
      const int p = k + PFP;
      for (int i = 4 * p + 1; i <= 4 * p + 4; ++i)
        if (i <= ilast) issue(i);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (!live_j) continue;
    const int r = rb + k;
    float v[5][5];
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const float* rr = ring + (size_t)((4 * k + a) % NSR) * kConv1RowLen;
      const float4 q = *reinterpret_cast<const float4*>(rr + 4 + 4 * t);
      v[a][0] = rr[3 + 4 * t];
      v[a][1] = q.x;
      v[a][2] = q.y;
      v[a][3] = q.z;
      v[a][4] = q.w;
    }
    auto row = [&](int h, const float (&v0)[5], const float (&v1)[5], const float (&v2)[5]) {
      const int p = 2 * r + h;
      if (p >= H1) return;
      const float* vr[3] = {v0, v1, v2};
      float o[2][8];
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const float ww = wr[k2 * 9 + a * 3 + b];
            s0 = fmaf(ww, vr[a][b], s0);
            s1 = fmaf(ww, vr[a][b + 2], s1);
          }
        o[0][k2] = fmaxf(s0, 0.f);
        o[1][k2] = fmaxf(s1, 0.f);
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
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

}  // namespace dagrt
