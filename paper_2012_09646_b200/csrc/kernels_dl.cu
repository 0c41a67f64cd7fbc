// Deep-learning (DL) kernels for sm_100a (§V-B; Fig. 6
// L702-710; architecture: DESIGN.md reading R-DL).  NHWC fp32,
// cross-correlation, zero padding, shared weights for both branches.
//
//   conv1: x (H x W x 1)   -> c1 (H1 x W1 x 8),  3x3 stride 2 pad 1, ReLU
//   pool : c1              -> p  (H1/2 x W1/2 x 8), 2x2 mean, stride 2
//   conv2: p (H2 x W2 x 8) -> c2 (H3 x W3 x 16), 3x3 stride 2 pad 1, ReLU
//   concat, dot (dense layer, one output)
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

// POOL: 2x2 mean, stride 2, 8 channels (two float4 per pixel).
__global__ void __launch_bounds__(256) k_pool(const float* __restrict__ in, float* __restrict__ out,
                                              int H1, int W1) {
  const int H2 = H1 / 2, W2 = W1 / 2;
  const long long total = (long long)H2 * W2 * 2;  // half-pixels (4 channels each)
  const float4* src = reinterpret_cast<const float4*>(in);
  float4* dst = reinterpret_cast<float4*>(out);
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < total;
       id += (long long)gridDim.x * blockDim.x) {
    const long long pix = id >> 1;
    const int h = (int)(id & 1);
    const int i = (int)(pix / W2), jj = (int)(pix % W2);
    const size_t r0 = ((size_t)(2 * i) * W1 + 2 * jj) * 2 + h;
    const size_t r1 = r0 + (size_t)W1 * 2;
    float4 a = ldg_stream(src + r0), b = ldg_stream(src + r0 + 2);
    float4 c = ldg_stream(src + r1), d = ldg_stream(src + r1 + 2);
    float4 o;
    o.x = 0.25f * (a.x + b.x + c.x + d.x);
    o.y = 0.25f * (a.y + b.y + c.y + d.y);
    o.z = 0.25f * (a.z + b.z + c.z + d.z);
    o.w = 0.25f * (a.w + b.w + c.w + d.w);
    dst[id] = o;
  }
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

// CONCAT: z = [a; b]
__global__ void __launch_bounds__(256) k_concat(const float* __restrict__ a,
                                                const float* __restrict__ b, float* __restrict__ z,
                                                long long na, long long nb) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  if (aligned16(a) && aligned16(b) && aligned16(z) && (na & 3) == 0 && (nb & 3) == 0) {
    const long long a4 = na >> 2, b4 = nb >> 2;
    const float4* A = reinterpret_cast<const float4*>(a);
    const float4* B = reinterpret_cast<const float4*>(b);
    float4* Z = reinterpret_cast<float4*>(z);
    for (long long i = tid; i < a4 + b4; i += nth) Z[i] = i < a4 ? ldg_stream(A + i) : ldg_stream(B + (i - a4));
  } else {
    for (long long i = tid; i < na + nb; i += nth) z[i] = i < na ? a[i] : b[i - na];
  }
}

// DOT (dense layer): r = sum_i z_i wd_i, fp64 accumulation, deterministic.
__global__ void __launch_bounds__(256) k_dot(const float* __restrict__ z,
                                             const float* __restrict__ wd, RedOut* r, long long n) {
  __shared__ double sh[32];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long long done = 0;
  if (aligned16(z) && aligned16(wd)) {
    const long long n4 = n >> 2;
    const float4* Z = reinterpret_cast<const float4*>(z);
    const float4* Wd = reinterpret_cast<const float4*>(wd);
    for (long long i = tid; i < n4; i += nth) {
      float4 a = ldg_stream(Z + i), b = ldg_stream(Wd + i);
      acc = fma((double)a.x, (double)b.x, acc);
      acc = fma((double)a.y, (double)b.y, acc);
      acc = fma((double)a.z, (double)b.z, acc);
      acc = fma((double)a.w, (double)b.w, acc);
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) acc = fma((double)z[i], (double)wd[i], acc);
  double blk = block_reduce(acc, OpAdd(), sh);
  double total;
  if (grid_finish(r, blk, OpAdd(), 0.0, &total, sh) && threadIdx.x == 0) r->result = (float)total;
}

// launch contracts (dagrt_launch validates them; builtin.h LaunchCheck)
static const char* v_conv1(const LaunchCheck& L) {  // x, w1, out, H, W
  const int H = L.i32(3), W = L.i32(4);
  if (H < 0 || W < 0) return "negative image size";
  const uint64_t h1 = (H + 1) / 2, w1 = (W + 1) / 2;
  if (!fits(L, 0, 4ull * H * W) || !fits(L, 1, 4 * 72) || !fits(L, 2, 32 * h1 * w1))
    return "x (4 H W), w1 (288) or out (32 ceil(H/2) ceil(W/2)) too small";
  return L.nthreads() == 256 ? nullptr : "256 threads per CTA";
}
static const char* v_pool(const LaunchCheck& L) {  // in, out, H1, W1 (8 channels)
  const int H = L.i32(2), W = L.i32(3);
  if (H < 0 || W < 0) return "negative size";
  if (!fits(L, 0, 32ull * H * W) || !fits(L, 1, 32ull * (H / 2) * (W / 2))) return "in / out too small";
  return L.nthreads() <= 256 ? nullptr : "at most 256 threads per CTA";
}
static const char* v_concat(const LaunchCheck& L) {  // a, b, z, na, nb
  const uint64_t na = (uint64_t)L.i(3), nb = (uint64_t)L.i(4);
  return fits(L, 0, 4 * na) && fits(L, 1, 4 * nb) && fits(L, 2, 4 * (na + nb)) ? nullptr : "arrays too small";
}
static const char* v_dot(const LaunchCheck& L) {  // z, wd, r, n
  const uint64_t n = (uint64_t)L.i(3);
  if (!fits(L, 0, 4 * n) || !fits(L, 1, 4 * n)) return "vectors need 4 n bytes";
  return check_reduction(L, 2);
}

static const Builtin kDl[] = {
    // one row per iteration, registers capped for 4 CTAs/SM (687 us vs 710 us uncapped)
    // product: two output rows per iteration, 3 CTAs/SM; grid.y walks row PAIRS
    // (633 us vs 690 us for one row per iteration, tools/conv2_variants.py)
    {"conv1", (const void*)k_conv1_r2b3, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, 0, nullptr, v_conv1},
    {"conv1_b3", (const void*)k_conv1_b3, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_b4", (const void*)k_conv1_b4, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_b4cs", (const void*)k_conv1_b4cs, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    // two output rows per iteration (grid.y walks row pairs)
    {"conv1_r2b3", (const void*)k_conv1_r2b3, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_r2b3cs", (const void*)k_conv1_r2b3cs, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_r2b2", (const void*)k_conv1_r2b2, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"conv1_b1", (const void*)k_conv1, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"pool", (const void*)k_pool, "const ptr, out ptr, sint32, sint32", KF_NONE, 0, nullptr, v_pool},
    // CUDA-core variant of the second convolution (the tcgen05 one is "conv2")
    {"conv2_ffma", (const void*)k_conv2, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE},
    {"concat", (const void*)k_concat, "const ptr, const ptr, out ptr, sint64, sint64", KF_NONE, 0, nullptr, v_concat},
    {"dot", (const void*)k_dot, "const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_dot},
};
DAGRT_REGISTER_BUILTINS(kDl);

}  // namespace dagrt
