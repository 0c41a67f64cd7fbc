// VEC and Black & Scholes kernels for sm_100a.
//
// VEC (§V-B; Fig. 4): square x2, then the sum of
// differences.  B&S (L865-870, adapted from the CUDA-samples pricer [28]):
// fp64 European call price per option.
#include "kcommon.cuh"

namespace dagrt {

// K1: x1[i] = x[i]^2 (out of place).  HBM-streaming: 128-bit loads and
// stores, grid-stride, 2 float4 in flight per thread per iteration.
__global__ void __launch_bounds__(256) k_square(const float* __restrict__ x, float* __restrict__ y,
                                                long long n) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(x) && aligned16(y)) {
    const long long n4 = n >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4* y4 = reinterpret_cast<float4*>(y);
    long long i = tid;
    for (; i + nth < n4; i += 2 * nth) {
      float4 a = ldg_stream(x4 + i), b = ldg_stream(x4 + i + nth);
      a.x *= a.x; a.y *= a.y; a.z *= a.z; a.w *= a.w;
      b.x *= b.x; b.y *= b.y; b.z *= b.z; b.w *= b.w;
      y4[i] = a;
      y4[i + nth] = b;
    }
    for (; i < n4; i += nth) {
      float4 a = ldg_stream(x4 + i);
      a.x *= a.x; a.y *= a.y; a.z *= a.z; a.w *= a.w;
      y4[i] = a;
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) {
    float v = x[i];
    y[i] = v * v;
  }
}

// K2: z = sum_i (x1[i] - y1[i]), fp64 accumulation, deterministic grid finish.
__global__ void __launch_bounds__(256) k_reduce_diff(const float* __restrict__ x1,
                                                     const float* __restrict__ y1, RedOut* z,
                                                     long long n) {
  __shared__ double sh[32];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long long done = 0;
  if (aligned16(x1) && aligned16(y1)) {
    const long long n4 = n >> 2;
    const float4* a4 = reinterpret_cast<const float4*>(x1);
    const float4* b4 = reinterpret_cast<const float4*>(y1);
    for (long long i = tid; i < n4; i += nth) {
      float4 a = ldg_stream(a4 + i), b = ldg_stream(b4 + i);
      acc += ((double)a.x - (double)b.x) + ((double)a.y - (double)b.y) +
             ((double)a.z - (double)b.z) + ((double)a.w - (double)b.w);
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) acc += (double)x1[i] - (double)y1[i];
  double blk = block_reduce(acc, OpAdd(), sh);
  double total;
  if (grid_finish(z, blk, OpAdd(), 0.0, &total, sh) && threadIdx.x == 0) z->result = (float)total;
}

}  // namespace dagrt

#include "bs_math.cuh"

namespace dagrt {

// ---------------------------------------------------------------- B&S product
// 37.5 FP64 ops per option (the lean pricer bs_price_l: 512-entry log and
// 128-entry exp tables), inputs streamed by cp.async.bulk into a 3-stage
// shared-memory ring, 6 options per thread in lockstep, 2 CTAs/SM one wave
// (bs2_tma_body, bs_math.cuh): 40.3 us per 10M options vs 41.6 for the same
// body with the round-2 pricer (bs2t_o6s3b2), tools/bs_variants.py.  The
// round-1 kernels and the other tuning variants are in exp/bs_variants.cu.
BS2L_VARIANT(k_bs2l_o6s3b2, 6, 3, 2)

// ---------------------------------------------------------------- B&S in fp32 (f4)
// The same pricing (A&S 26.2.17 CND) in fp32 storage and
// arithmetic: 8 bytes per option instead of 16 and no FP64 pipe, so the kernel
// is HBM-bound ("fp32 B&S variant, HBM-bound instead of
// FP64-bound").  Accuracy is fp32's (checked against the fp64 oracle with the
// north_star's fp32 criterion, 1e-4 |o| + 1e-4 rms(o)).  4 options per thread
// with 128-bit loads/stores, grid-stride.
// Same algebra as the fp64 pricer: one exponential per option (phi(d2) =
// phi(d1) S e^{RT}/K), the hardware approximations (MUFU lg2 / ex2 / rcp,
// ~2^-21 relative) that fp32's criterion allows, constants hoisted per CTA:
// ~35 instructions per option, so the kernel is HBM-bound (the first fp32
// version with IEEE divisions and the accurate logf/expf issued ~150 per
// option and ran at 0.25 of HBM).
struct BsF32C {
  float inv_k, inv_vst, mu_s, vst, kexp, c2;
};
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float bs_price_f32(float s, const BsF32C& C) {
  const float A = 0.2316419f, R2PI = 0.39894228040143268f;
  const float d1 = fmaf(__logf(s * C.inv_k), C.inv_vst, C.mu_s);
  const float d2 = d1 - C.vst;
  const float phi1 = R2PI * __expf(-0.5f * d1 * d1);
  const float phi2 = phi1 * (s * C.c2);
  const float k1 = rcp_approx(fmaf(A, fabsf(d1), 1.f)), k2 = rcp_approx(fmaf(A, fabsf(d2), 1.f));
  const float q1 = k1 * fmaf(k1, fmaf(k1, fmaf(k1, fmaf(k1, 1.330274429f, -1.821255978f), 1.781477937f), -0.356563782f),
                             0.31938153f);
  const float q2 = k2 * fmaf(k2, fmaf(k2, fmaf(k2, fmaf(k2, 1.330274429f, -1.821255978f), 1.781477937f), -0.356563782f),
                             0.31938153f);
  const float p1 = phi1 * q1, p2 = phi2 * q2;
  const float c1 = d1 > 0.f ? 1.f - p1 : p1, cc2 = d2 > 0.f ? 1.f - p2 : p2;
  return fmaf(s, c1, -C.kexp * cc2);
}

__global__ void __launch_bounds__(256) k_bs_f32(const float* __restrict__ s, float* __restrict__ c, long long n,
                                                float r, float v, float t, float k) {
  BsF32C C;
  C.vst = v * sqrtf(t);
  C.inv_vst = 1.f / C.vst;
  C.mu_s = (r + 0.5f * v * v) * t / C.vst;
  C.inv_k = 1.f / k;
  C.kexp = k * expf(-r * t);
  C.c2 = expf(r * t) / k;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(s) && aligned16(c)) {
    // two 16-byte loads in flight per thread before any use (the one-load
    // loop was latency-bound at 0.49 of HBM)
    const long long n4 = n >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(s);
    float4* c4 = reinterpret_cast<float4*>(c);
    long long i = tid;
    for (; i + nth < n4; i += 2 * nth) {
      const float4 x = ldg_stream(s4 + i), y = ldg_stream(s4 + i + nth);
      c4[i] = make_float4(bs_price_f32(x.x, C), bs_price_f32(x.y, C), bs_price_f32(x.z, C), bs_price_f32(x.w, C));
      c4[i + nth] =
          make_float4(bs_price_f32(y.x, C), bs_price_f32(y.y, C), bs_price_f32(y.z, C), bs_price_f32(y.w, C));
    }
    if (i < n4) {
      const float4 x = ldg_stream(s4 + i);
      c4[i] = make_float4(bs_price_f32(x.x, C), bs_price_f32(x.y, C), bs_price_f32(x.z, C), bs_price_f32(x.w, C));
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) c[i] = bs_price_f32(s[i], C);
}

// launch contracts (dagrt_launch validates them; builtin.h LaunchCheck)
static const char* v_square(const LaunchCheck& L) {
  const uint64_t n = (uint64_t)L.i(2);
  return fits(L, 0, 4 * n) && fits(L, 1, 4 * n) ? nullptr : "x and x1 need 4 n bytes";
}
static const char* v_reduce_diff(const LaunchCheck& L) {
  const uint64_t n = (uint64_t)L.i(3);
  if (!fits(L, 0, 4 * n) || !fits(L, 1, 4 * n)) return "inputs need 4 n bytes";
  return check_reduction(L, 2);
}
static const char* v_bs_f32(const LaunchCheck& L) {
  const uint64_t n = (uint64_t)L.i(2);
  return fits(L, 0, 4 * n) && fits(L, 1, 4 * n) ? nullptr : "prices and calls need 4 n bytes";
}
static const char* v_bs(const LaunchCheck& L) {
  const uint64_t n = (uint64_t)L.i(2);
  if (!fits(L, 0, 8 * n) || !fits(L, 1, 8 * n)) return "prices and calls need 8 n bytes";
  return L.nthreads() <= 256 ? nullptr : "at most 256 threads per CTA";
}
static const Builtin kVecBs[] = {
    {"square", (const void*)k_square, "const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_square},
    {"reduce_diff", (const void*)k_reduce_diff, "const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_reduce_diff},
    // product: lean loop, 3 pairs per thread, 2 CTAs/SM, one wave (44.8 us per
    // 10M options vs 46.2 for 4 pairs (k_bs_l4b2) in three back-to-back runs,
    // 49.5 for k_bs, tools/bs_variants.py); k_bs kept as "bs_p4"
    // product (round 2): 37.5 FP64 ops per option (lean algebraic pricer),
    // inputs streamed by cp.async.bulk into a 3-stage ring, 6 options per
    // thread in lockstep, 2 CTAs/SM one wave: 40.3 us per 10M options vs 45.8
    // for the round-1 product (bs_l3b2), tools/bs_variants.py
    {"bs", (const void*)k_bs2l_o6s3b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, 0,
     nullptr, v_bs},
    // f4: the same pricing in fp32 (HBM-bound)
    {"bs_f32", (const void*)k_bs_f32, "const ptr, out ptr, sint64, float, float, float, float", KF_NONE, 0, nullptr,
     v_bs_f32},
};
DAGRT_REGISTER_BUILTINS(kVecBs);

}  // namespace dagrt
