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

// ---------------------------------------------------------------- B&S
// A&S 26.2.17 cumulative normal, fp64 (L868-869: double precision).
__device__ __forceinline__ double cnd(double d) {
  const double A1 = 0.31938153, A2 = -0.356563782, A3 = 1.781477937, A4 = -1.821255978,
               A5 = 1.330274429, RSQRT2PI = 0.39894228040143267794;
  double k = 1.0 / (1.0 + 0.2316419 * fabs(d));
  double p = RSQRT2PI * exp(-0.5 * d * d) * (k * (A1 + k * (A2 + k * (A3 + k * (A4 + k * A5)))));
  return d > 0 ? 1.0 - p : p;
}

__device__ __forceinline__ double bs_price(double s, double k, double r, double v, double t) {
  const double sqrt_t = sqrt(t);
  const double d1 = (log(s / k) + (r + 0.5 * v * v) * t) / (v * sqrt_t);
  const double d2 = d1 - v * sqrt_t;
  return s * cnd(d1) - k * exp(-r * t) * cnd(d2);
}

// K3: c[i] = BlackScholesCall(s[i]; K, R, V, T), 128-bit fp64 loads.
__global__ void __launch_bounds__(256) k_bs(const double* __restrict__ s, double* __restrict__ c,
                                            long long n, double r, double v, double t, double k) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(s) && aligned16(c)) {
    const long long n2 = n >> 1;
    const double2* s2 = reinterpret_cast<const double2*>(s);
    double2* c2 = reinterpret_cast<double2*>(c);
    for (long long i = tid; i < n2; i += nth) {
      double2 x = ldg_stream(s2 + i);
      double2 y;
      y.x = bs_price(x.x, k, r, v, t);
      y.y = bs_price(x.y, k, r, v, t);
      c2[i] = y;
    }
    done = n2 << 1;
  }
  for (long long i = done + tid; i < n; i += nth) c[i] = bs_price(s[i], k, r, v, t);
}

static const Builtin kVecBs[] = {
    {"square", (const void*)k_square, "const ptr, out ptr, sint64", KF_NONE},
    {"reduce_diff", (const void*)k_reduce_diff, "const ptr, const ptr, out ptr, sint64", KF_NONE},
    {"bs", (const void*)k_bs, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
};
DAGRT_REGISTER_BUILTINS(kVecBs);

}  // namespace dagrt
