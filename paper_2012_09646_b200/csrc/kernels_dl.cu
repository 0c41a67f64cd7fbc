// Deep-learning (DL) kernels for sm_100a (§V-B; Fig. 6
// L702-710; architecture: DESIGN.md reading R-DL).  NHWC fp32,
// cross-correlation, zero padding, shared weights for both branches.
//
//   conv1: x (H x W x 1)   -> c1 (H1 x W1 x 8),  3x3 stride 2 pad 1, ReLU
//   pool : c1              -> p  (H1/2 x W1/2 x 8), 2x2 mean, stride 2
//   conv2: p (H2 x W2 x 8) -> c2 (H3 x W3 x 16), 3x3 stride 2 pad 1, ReLU
//   concat, dot (dense layer, one output)
#include "conv1.cuh"

namespace dagrt {

// product conv1: two output rows per iteration, 3 CTAs/SM; grid.y walks row
// PAIRS (633 us vs 690 us for one row per iteration, tools/conv2_variants.py);
// outputs transposed per warp through shared memory so that each 128-bit
// store covers 512 contiguous bytes, with the evict-first policy (598 vs
// 630 us, 0.82 vs 0.78 of HBM, bitwise-identical: tools/conv1_variants.py,
// profiles/r2_conv1_variants.json); the other shapes are in exp/dl_variants.cu
__global__ void __launch_bounds__(256, 3) k_conv1_r2b3(const float* __restrict__ x, const float* __restrict__ w,
                                                       float* __restrict__ out, int H, int W) {
  conv1_body2<true, true>(x, w, out, H, W);
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
    auto dp = [](float4 a, float4 b, double t) {
      t = fma((double)a.x, (double)b.x, t);
      t = fma((double)a.y, (double)b.y, t);
      t = fma((double)a.z, (double)b.z, t);
      return fma((double)a.w, (double)b.w, t);
    };
    double acc1 = 0.0;
    long long i = tid;
    for (; i + nth < n4; i += 2 * nth) {  // four 16-byte loads in flight, two chains
      const float4 a = ldg_stream(Z + i), b = ldg_stream(Wd + i), c = ldg_stream(Z + i + nth),
                   d = ldg_stream(Wd + i + nth);
      acc = dp(a, b, acc);
      acc1 = dp(c, d, acc1);
    }
    for (; i < n4; i += nth) acc = dp(ldg_stream(Z + i), ldg_stream(Wd + i), acc);
    acc += acc1;
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
    {"conv1", (const void*)k_conv1_r2b3, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, 0, nullptr, v_conv1},
    {"pool", (const void*)k_pool, "const ptr, out ptr, sint32, sint32", KF_NONE, 0, nullptr, v_pool},
    {"concat", (const void*)k_concat, "const ptr, const ptr, out ptr, sint64, sint64", KF_NONE, 0, nullptr, v_concat},
    {"dot", (const void*)k_dot, "const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_dot},
};
DAGRT_REGISTER_BUILTINS(kDl);

}  // namespace dagrt
