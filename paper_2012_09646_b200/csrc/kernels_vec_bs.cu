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
// fp64 throughout (L868-869).  A straightforward port (log, two exp, two
// divisions through libdevice) costs ~180 FP64 instructions per option and
// runs at 1/4 of the HBM roofline on B200 (FP64 pipe: 64 DFMA/clk/SM).  This
// version needs ~50:
//   * exp(-d2^2/2) = exp(-d1^2/2) * (S/K) * e^{RT}   (since d1 V sqrt(T) =
//     ln(S/K) + (R + V^2/2) T), so one exp per option instead of two;
//   * both A&S reciprocals 1/(1+a|d|) from ONE reciprocal of their product;
//   * table-driven log (128 entries, |r| <= 1/256, degree-5 series) and exp
//     (2^(j/64) table, |r| <= ln2/128, degree-5 Taylor) with the tables in
//     shared memory (lane-divergent indices would serialise constant memory);
//   * the 1/sqrt(2 pi) factor folded into the A&S coefficients.
// Each step is accurate to a few ulp; the result matches the fp64 oracle
// (libm) to ~1e-15 relative (tolerance 1e-10 rel + 1e-12 abs).
struct BsTables {
  double inv[128];    // 1 / (1 + (j + 0.5)/128)
  double lninv[128];  // -ln(inv[j])
  double exp2j[64];   // 2^(j/64)
};

constexpr double kRound = 6755399441055744.0;           // 1.5 * 2^52 (low word 0: an immediate)
// Constants whose low 32 bits are not zero live in the constant bank: DFMA
// and DMUL read a c[][] operand directly, whereas a literal would be
// rematerialised with two register moves per use inside the loop.
enum { kcThird, kcLn2, kc64Ln2, kcNegLn2_64Hi, kcNegLn2_64Lo, kc24th, kc6th, kcB1, kcB2, kcB3, kcB4, kcB5,
       kcA, kcCount };
__constant__ double kBsK[kcCount] = {
    1.0 / 3.0,
    0.6931471805599453,       // ln 2
    92.33248261689366,        // 64 / ln 2
    -0.01083042469326756,     // -(ln2/64), 32 significant bits
    -2.9815858269852933e-12,  // -(ln2/64 - hi)
    1.0 / 24.0,
    1.0 / 6.0,
    // A&S 26.2.17 coefficients times 1/sqrt(2 pi), and its p = 0.2316419
    0.1274147958962986, -0.1422483682996393, 0.7107068706716199, -0.7265760130580615,
    0.5307027142649737, 0.2316419};

__device__ __forceinline__ void bs_tables_init(BsTables& T) {
  for (int j = threadIdx.x; j < 128; j += blockDim.x) {
    const double c = 1.0 / (1.0 + (j + 0.5) / 128.0);
    T.inv[j] = c;
    T.lninv[j] = -log(c);
    if (j < 64) T.exp2j[j] = exp2(j / 64.0);
  }
  __syncthreads();
}

// ln(x), x positive normal: x = m 2^e, m in [1,2); ln x = e ln2 - ln c_j + ln(1 + r)
__device__ __forceinline__ double bs_log(double x, const BsTables& T) {
  const int hi = __double2hiint(x), lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const int j = (hi >> 13) & 127;
  const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, lo);
  const double r = fma(m, T.inv[j], -1.0);
  // ln(1+r) to r^4: |r| <= 1/256, the dropped r^5/5 is < 2e-13 absolute
  double p = fma(r, -0.25, kBsK[kcThird]);
  p = fma(r, p, -0.5);
  p = fma(r, p, 1.0);
  return fma((double)e, kBsK[kcLn2], fma(p, r, T.lninv[j]));
}

// exp(y) for y <= 0 (0 below about -700, where it is < 1e-304); the range
// test is an integer compare of the high word (keeps it off the FP64 pipe)
__device__ __forceinline__ double bs_exp(double y, const BsTables& T) {
  if ((__double2hiint(y) & 0x7fffffff) > 0x4085E000) return 0.0;
  const double t = fma(y, kBsK[kc64Ln2], kRound);
  const int n = __double2loint(t);
  const double nd = t - kRound;
  double r = fma(nd, kBsK[kcNegLn2_64Hi], y);
  r = fma(nd, kBsK[kcNegLn2_64Lo], r);
  // e^r to r^4: |r| <= ln2/128, the dropped r^5/120 is < 4e-14 relative
  double p = fma(r, kBsK[kc24th], kBsK[kc6th]);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = fma(r, p, 1.0);
  const double s = T.exp2j[n & 63] * p;
  return __hiloint2double(__double2hiint(s) + ((n >> 6) << 20), __double2loint(s));
}

struct BsConst {
  double mu_s;     // (R + V^2/2) T / (V sqrt T)
  double inv_vst;  // 1 / (V sqrt T)
  double vst;      // V sqrt T
  double inv_k;    // 1 / K
  double c2;       // e^{RT} / K
  double kexp;     // K e^{-RT}
};

__device__ __forceinline__ double bs_price(double s, const BsConst& C, const BsTables& T) {
  const double B1 = kBsK[kcB1], B2 = kBsK[kcB2], B3 = kBsK[kcB3], B4 = kBsK[kcB4], B5 = kBsK[kcB5],
               A = kBsK[kcA];
  const double L = bs_log(s * C.inv_k, T);
  const double d1 = fma(L, C.inv_vst, C.mu_s);
  const double d2 = d1 - C.vst;
  const double e1 = bs_exp(-0.5 * (d1 * d1), T);  // exp(-d1^2/2)
  const double e2 = e1 * (s * C.c2);                // exp(-d2^2/2)
  const double D1 = fma(A, fabs(d1), 1.0), D2 = fma(A, fabs(d2), 1.0);
  const double P = D1 * D2;
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(P));
  // one Newton step on the ~2^-23 hardware estimate: ~2^-46 relative
  const double er = fma(-P, y, 1.0);
  y = fma(y, er, y);
  const double k1 = D2 * y, k2 = D1 * y;
  double q1 = fma(k1, B5, B4);
  q1 = fma(k1, q1, B3);
  q1 = fma(k1, q1, B2);
  q1 = fma(k1, q1, B1);
  double q2 = fma(k2, B5, B4);
  q2 = fma(k2, q2, B3);
  q2 = fma(k2, q2, B2);
  q2 = fma(k2, q2, B1);
  const double p1 = (q1 * k1) * e1, p2 = (q2 * k2) * e2;
  // CND = d > 0 ? 1 - p : p, with the sign test on the high word (integer pipe)
  const double c1 = __double2hiint(d1) > 0 ? 1.0 - p1 : p1;
  const double c2 = __double2hiint(d2) > 0 ? 1.0 - p2 : p2;
  return fma(s, c1, -C.kexp * c2);
}

// ---------------------------------------------------------------- B&S, round 2
// Same A&S 26.2.17 pricing (SURVEY §8(c2) B&S), ~38 FP64 operations per
// option instead of 46, by algebra rather than approximation:
//   * C = S CND(d1) - K e^{-RT} CND(d2) with CND(d) = u + sigma p, u = [d > 0],
//     sigma = -1 if d > 0 else +1, p = phi(d) k poly(k):
//       K e^{-RT} p2 = K e^{-RT} phi(d2) w2 = S phi(d1) w2   (phi(d2) = phi(d1) S e^{RT}/K)
//     so C = (S u1 - K e^{-RT} u2) + S phi(d1) (sigma1 w1 - sigma2 w2): no
//     second exponential, no products by e2, the signs flipped on the integer
//     pipe (sign bit of w), the first term selected among {0, S, S - Ke^{-RT}}
//     (d2 < d1, so u2 implies u1);
//   * phi(d1) = exp(-h/2), h = d1^2: the -1/2 is folded into the exp's range
//     reduction and polynomial (r2 = h + 2 n ln2/64, e^{-r2/2} by a
//     polynomial in r2 with rescaled coefficients);
//   * exp reduction with one ln2/64 constant (error <= 745 * 2^-53 relative
//     ~ 1e-13, far inside the 1e-10 tolerance) instead of a hi/lo pair.
// The computation is written W options in lockstep (every statement over a
// small array), so independent FP64 chains interleave in the instruction
// stream whatever ptxas's scheduler does with the inlined copies.
enum { kc2Ln2_64, kcNeg32Ln2, kcE0, kcE1, kcE2, kcE3, kcE4, kc2Count };
__constant__ double kBs2K[kc2Count] = {
    0.02166084939249829,      // 2 ln2 / 64
    -46.16624130844683,       // -32 / ln2  (t = round(-h/2 * 64/ln2))
    // e^{-r2/2} = 1 - r2/2 + r2^2/8 - r2^3/48 + r2^4/384 (|r2| <= 2 ln2/128)
    1.0 / 384.0, -1.0 / 48.0, 1.0 / 8.0, -0.5, 1.0};

template <int W>
__device__ __forceinline__ void bs_price_w(const double (&s)[W], double (&out)[W], const BsConst& C,
                                           const BsTables& T) {
  const double B1 = kBsK[kcB1], B2 = kBsK[kcB2], B3 = kBsK[kcB3], B4 = kBsK[kcB4], B5 = kBsK[kcB5],
               A = kBsK[kcA];
  double L[W];
#pragma unroll
  for (int w = 0; w < W; ++w) L[w] = bs_log(s[w] * C.inv_k, T);
  double d1[W], d2[W], h[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    d1[w] = fma(L[w], C.inv_vst, C.mu_s);
    d2[w] = d1[w] - C.vst;
    h[w] = d1[w] * d1[w];
  }
  // phi(d1) * sqrt(2 pi) = exp(-h/2), h clamped to ~1400 by an integer min on
  // its high word (exp(-700) ~ 1e-304 then stands for 0: the scaling by
  // 2^(n/64) stays in the normal range, and S e1 m is ~1e-298 or less)
  double e1[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const double hc = __hiloint2double(min(__double2hiint(h[w]), 0x4095E000), __double2loint(h[w]));
    const double t = fma(hc, kBs2K[kcNeg32Ln2], kRound);
    const int n = __double2loint(t);
    const double nd = t - kRound;
    const double r2 = fma(nd, kBs2K[kc2Ln2_64], hc);
    double p = fma(r2, kBs2K[kcE0], kBs2K[kcE1]);
    p = fma(r2, p, kBs2K[kcE2]);
    p = fma(r2, p, kBs2K[kcE3]);
    p = fma(r2, p, kBs2K[kcE4]);
    const double sc = T.exp2j[n & 63] * p;
    e1[w] = __hiloint2double(__double2hiint(sc) + ((n >> 6) << 20), __double2loint(sc));
  }
  double k1[W], k2[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const double D1 = fma(A, fabs(d1[w]), 1.0), D2 = fma(A, fabs(d2[w]), 1.0);
    const double P = D1 * D2;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(P));
    const double er = fma(-P, y, 1.0);
    y = fma(y, er, y);
    k1[w] = D2 * y;
    k2[w] = D1 * y;
  }
#pragma unroll
  for (int w = 0; w < W; ++w) {
    double q1 = fma(k1[w], B5, B4), q2 = fma(k2[w], B5, B4);
    q1 = fma(k1[w], q1, B3);
    q2 = fma(k2[w], q2, B3);
    q1 = fma(k1[w], q1, B2);
    q2 = fma(k2[w], q2, B2);
    q1 = fma(k1[w], q1, B1);
    q2 = fma(k2[w], q2, B1);
    const double w1 = q1 * k1[w], w2 = q2 * k2[w];
    const bool u1 = __double2hiint(d1[w]) > 0, u2 = __double2hiint(d2[w]) > 0;
    // sigma1 w1 - sigma2 w2: sign bits flipped on the integer pipe
    const double a1 = __hiloint2double(__double2hiint(w1) ^ (u1 ? 0x80000000 : 0), __double2loint(w1));
    const double a2 = __hiloint2double(__double2hiint(w2) ^ (u2 ? 0 : 0x80000000), __double2loint(w2));
    const double m = a1 + a2;
    const double sk = s[w] - C.kexp;
    const double base = u2 ? sk : (u1 ? s[w] : 0.0);
    out[w] = fma(s[w] * e1[w], m, base);
  }
}

// Lean loop of bs_body_lean with the lockstep pricer: PAIRS double2 per
// thread per group, priced W options at a time.
template <int PAIRS, int W>
__device__ __forceinline__ void bs2_body(const double* __restrict__ s, double* __restrict__ c, long long n,
                                         double r, double v, double t, double k) {
  __shared__ BsTables T;
  bs_tables_init(T);
  BsConst C;
  const double vst = v * sqrt(t);
  C.vst = vst;
  C.inv_vst = 1.0 / vst;
  C.mu_s = (r + 0.5 * v * v) * t / vst;
  C.inv_k = 1.0 / k;
  C.c2 = exp(r * t) / k;
  C.kexp = k * exp(-r * t);
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned nth = gridDim.x * blockDim.x;
  if (!(aligned16(s) && aligned16(c)) || n >= (1ll << 31)) {
    for (long long i = tid; i < n; i += nth) {
      double a[1] = {s[i]}, o[1];
      bs_price_w<1>(a, o, C, T);
      c[i] = o[0];
    }
    return;
  }
  static_assert((2 * PAIRS) % W == 0 && W % 2 == 0, "W even, dividing the options per group");
  const unsigned n2 = (unsigned)(n >> 1);
  const unsigned step = PAIRS * nth;
  const unsigned nfull = n2 / step;
  const double2* s2 = reinterpret_cast<const double2*>(s);
  double2* c2 = reinterpret_cast<double2*>(c);
  double2 xa[PAIRS], xb[PAIRS];
  auto load = [&](double2(&x)[PAIRS], unsigned base) {
#pragma unroll
    for (int q = 0; q < PAIRS; ++q) x[q] = ldg_stream(s2 + base + q * nth);
  };
  auto price = [&](const double2(&x)[PAIRS], unsigned base) {
#pragma unroll
    for (int g0 = 0; g0 < 2 * PAIRS; g0 += W) {
      double a[W], o[W];
#pragma unroll
      for (int w = 0; w < W; ++w) a[w] = ((g0 + w) & 1) ? x[(g0 + w) >> 1].y : x[(g0 + w) >> 1].x;
      bs_price_w<W>(a, o, C, T);
#pragma unroll
      for (int w = 0; w < W; w += 2) c2[base + ((g0 + w) >> 1) * nth] = make_double2(o[w], o[w + 1]);
    }
  };
  unsigned base = tid, j = 0;
  if (nfull > 0) load(xa, base);
  for (; j + 2 <= nfull; j += 2) {
    load(xb, base + step);
    price(xa, base);
    if (j + 2 < nfull) load(xa, base + 2 * step);
    price(xb, base + step);
    base += 2 * step;
  }
  if (j < nfull) {
    price(xa, base);
    base += step;
  }
#pragma unroll
  for (int q = 0; q < PAIRS; ++q) {  // tail: the last partial group
    const unsigned i = base + q * nth;
    if (i < n2) {
      const double2 x = ldg_stream(s2 + i);
      double a[2] = {x.x, x.y}, o[2];
      bs_price_w<2>(a, o, C, T);
      c2[i] = make_double2(o[0], o[1]);
    }
  }
  if ((n & 1) && tid == 0) {
    double a[1] = {s[n - 1]}, o[1];
    bs_price_w<1>(a, o, C, T);
    c[n - 1] = o[0];
  }
}
#define BS2_VARIANT(NAME, PAIRS, W, MINB)                                                         \
  __global__ void __launch_bounds__(256, MINB) NAME(const double* __restrict__ s,                 \
                                                    double* __restrict__ c, long long n, double r, \
                                                    double v, double t, double k) {                \
    bs2_body<PAIRS, W>(s, c, n, r, v, t, k);                                                       \
  }
BS2_VARIANT(k_bs2_p3w2b2, 3, 2, 2)
BS2_VARIANT(k_bs2_p2w2b3, 2, 2, 3)
BS2_VARIANT(k_bs2_p2w4b2, 2, 4, 2)
BS2_VARIANT(k_bs2_p4w2b2, 4, 2, 2)
BS2_VARIANT(k_bs2_p1w2b4, 1, 2, 4)

// TMA-staged form: each CTA walks contiguous chunks of 256 * OPT options;
// one thread streams chunk k + STAGES into a shared-memory ring with a bulk
// copy (cp.async.bulk, completion on an mbarrier) while the CTA prices chunk
// k -- deep prefetch at no register cost (the register-prefetched loops were
// long-scoreboard bound: ncu, profiles/).  Each thread prices OPT options of a
// chunk in lockstep, reading them with 128-bit shared loads; the prices go
// straight to global memory (coalesced 16-byte stores).
__device__ __forceinline__ void bs_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void bs_mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bs_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}

template <int OPT, int STAGES>
__device__ __forceinline__ void bs2_tma_body(const double* __restrict__ s, double* __restrict__ c, long long n,
                                             double r, double v, double t, double k) {
  constexpr int kChunk = 256 * OPT;  // options per chunk (blockDim.x == 256)
  __shared__ BsTables T;
  __shared__ __align__(128) double ring[STAGES][kChunk];
  __shared__ uint64_t full[STAGES];
  bs_tables_init(T);
  BsConst C;
  const double vst = v * sqrt(t);
  C.vst = vst;
  C.inv_vst = 1.0 / vst;
  C.mu_s = (r + 0.5 * v * v) * t / vst;
  C.inv_k = 1.0 / k;
  C.c2 = exp(r * t) / k;
  C.kexp = k * exp(-r * t);
  const int tid = threadIdx.x;
  if (!(aligned16(s) && aligned16(c)) || blockDim.x != 256) {
    for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < n; i += (long long)gridDim.x * blockDim.x) {
      double a[2] = {s[i], 1.0}, o[2];
      bs_price_w<2>(a, o, C, T);
      c[i] = o[0];
    }
    return;
  }
  const long long nfullc = n / kChunk;  // whole chunks via the ring; the tail directly
  const long long G = gridDim.x;
  if (tid == 0) {
    for (int q = 0; q < STAGES; ++q) bs_mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < STAGES; ++q) {
      const long long ch = blockIdx.x + q * G;
      if (ch < nfullc) bs_bulk_g2s(ring[q], s + ch * kChunk, kChunk * 8, &full[q]);
    }
  int it = 0;
  for (long long ch = blockIdx.x; ch < nfullc; ch += G, ++it) {
    const int st = it % STAGES;
    bs_mbar_wait(&full[st], (unsigned)((it / STAGES) & 1));
    double a[OPT], o[OPT];
#pragma unroll
    for (int q = 0; q < OPT / 2; ++q) {  // options 2 (tid + 256 q) and +1: 16-byte shared loads
      const double2 x = reinterpret_cast<const double2*>(ring[st])[tid + 256 * q];
      a[2 * q] = x.x;
      a[2 * q + 1] = x.y;
    }
    __syncthreads();  // every thread has its options: the stage may be refilled
    if (tid == 0 && ch + STAGES * G < nfullc) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bs_bulk_g2s(ring[st], s + (ch + STAGES * G) * kChunk, kChunk * 8, &full[st]);
    }
    bs_price_w<OPT>(a, o, C, T);
    double2* dst = reinterpret_cast<double2*>(c + ch * kChunk);
#pragma unroll
    for (int q = 0; q < OPT / 2; ++q) dst[tid + 256 * q] = make_double2(o[2 * q], o[2 * q + 1]);
  }
  for (long long i = nfullc * kChunk + (long long)blockIdx.x * blockDim.x + tid; i < n; i += G * blockDim.x) {
    double a[2] = {s[i], 1.0}, o[2];
    bs_price_w<2>(a, o, C, T);
    c[i] = o[0];
  }
}
#define BS2T_VARIANT(NAME, OPT, STAGES, MINB)                                                      \
  __global__ void __launch_bounds__(256, MINB) NAME(const double* __restrict__ s,                 \
                                                    double* __restrict__ c, long long n, double r, \
                                                    double v, double t, double k) {                \
    bs2_tma_body<OPT, STAGES>(s, c, n, r, v, t, k);                                                \
  }
BS2T_VARIANT(k_bs2t_o4s4b2, 4, 4, 2)
BS2T_VARIANT(k_bs2t_o4s3b3, 4, 3, 3)
BS2T_VARIANT(k_bs2t_o2s4b4, 2, 4, 4)
BS2T_VARIANT(k_bs2t_o6s3b2, 6, 3, 2)

// ---------------------------------------------------------------- B&S in fp32 (f4)
// The same pricing (A&S 26.2.17 CND) in fp32 storage and
// arithmetic: 8 bytes per option instead of 16 and no FP64 pipe, so the kernel
// is HBM-bound ("fp32 B&S variant, HBM-bound instead of
// FP64-bound").  Accuracy is fp32's (checked against the fp64 oracle with the
// north_star's fp32 criterion, 1e-4 |o| + 1e-4 rms(o)).  4 options per thread
// with 128-bit loads/stores, grid-stride.
__device__ __forceinline__ float bs_price_f32(float s, float r, float v, float t, float k) {
  const float vst = v * sqrtf(t);
  const float d1 = (logf(s / k) + (r + 0.5f * v * v) * t) / vst;
  const float d2 = d1 - vst;
  auto cnd = [](float d) {
    const float kk = 1.f / fmaf(0.2316419f, fabsf(d), 1.f);
    const float p = 0.39894228040143268f * expf(-0.5f * d * d) * kk *
                    fmaf(kk, fmaf(kk, fmaf(kk, fmaf(kk, 1.330274429f, -1.821255978f), 1.781477937f), -0.356563782f),
                         0.31938153f);
    return d > 0.f ? 1.f - p : p;
  };
  return s * cnd(d1) - k * expf(-r * t) * cnd(d2);
}
__global__ void __launch_bounds__(256) k_bs_f32(const float* __restrict__ s, float* __restrict__ c, long long n,
                                                float r, float v, float t, float k) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(s) && aligned16(c)) {
    const long long n4 = n >> 2;
    for (long long i = tid; i < n4; i += nth) {
      const float4 x = ldg_stream(reinterpret_cast<const float4*>(s) + i);
      reinterpret_cast<float4*>(c)[i] = make_float4(bs_price_f32(x.x, r, v, t, k), bs_price_f32(x.y, r, v, t, k),
                                                    bs_price_f32(x.z, r, v, t, k), bs_price_f32(x.w, r, v, t, k));
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) c[i] = bs_price_f32(s[i], r, v, t, k);
}

// K3: c[i] = BlackScholesCall(s[i]; K, R, V, T), 128-bit fp64 loads/stores.
// PAIRS double2 per thread per iteration (independent chains for the FP64
// pipe to interleave); the next group's loads are issued before pricing.
template <int PAIRS>
__device__ __forceinline__ void bs_body(const double* __restrict__ s, double* __restrict__ c,
                                        long long n, double r, double v, double t, double k) {
  __shared__ BsTables T;
  bs_tables_init(T);
  BsConst C;
  const double vst = v * sqrt(t);
  C.vst = vst;
  C.inv_vst = 1.0 / vst;
  C.mu_s = (r + 0.5 * v * v) * t / vst;
  C.inv_k = 1.0 / k;
  C.c2 = exp(r * t) / k;
  C.kexp = k * exp(-r * t);
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(s) && aligned16(c)) {
    const long long n2 = n >> 1;
    const double2* s2 = reinterpret_cast<const double2*>(s);
    double2* c2 = reinterpret_cast<double2*>(c);
    double2 x[PAIRS];
#pragma unroll
    for (int q = 0; q < PAIRS; ++q) {
      const long long i = tid + q * nth;
      x[q] = i < n2 ? ldg_stream(s2 + i) : make_double2(1.0, 1.0);
    }
    for (long long i0 = tid; i0 < n2; i0 += PAIRS * nth) {
      double2 nx[PAIRS];
#pragma unroll
      for (int q = 0; q < PAIRS; ++q) {
        const long long i = i0 + (PAIRS + q) * nth;
        nx[q] = i < n2 ? ldg_stream(s2 + i) : x[q];
      }
#pragma unroll
      for (int q = 0; q < PAIRS; ++q) {
        const long long i = i0 + q * nth;
        double2 y;
        y.x = bs_price(x[q].x, C, T);
        y.y = bs_price(x[q].y, C, T);
        if (i < n2) c2[i] = y;
        x[q] = nx[q];
      }
    }
    done = n2 << 1;
  }
  for (long long i = done + tid; i < n; i += nth) c[i] = bs_price(s[i], C, T);
}

// Lean form of bs_body: 32-bit pair indices, no bounds tests in the main
// loop (full groups first, then one checked tail), and two register buffers
// used in turn (load group j+1 into one while the other is priced) instead of
// copying the prefetched group into the working one -- the integer
// bookkeeping of the 64-bit, per-pair-checked loop was ~10 of the ~100 issue
// slots per option (SASS of k_bs_p4b2).  Same arithmetic and results.
template <int PAIRS>
__device__ __forceinline__ void bs_body_lean(const double* __restrict__ s, double* __restrict__ c,
                                             long long n, double r, double v, double t, double k) {
  __shared__ BsTables T;
  bs_tables_init(T);
  BsConst C;
  const double vst = v * sqrt(t);
  C.vst = vst;
  C.inv_vst = 1.0 / vst;
  C.mu_s = (r + 0.5 * v * v) * t / vst;
  C.inv_k = 1.0 / k;
  C.c2 = exp(r * t) / k;
  C.kexp = k * exp(-r * t);
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned nth = gridDim.x * blockDim.x;
  if (!(aligned16(s) && aligned16(c)) || n >= (1ll << 31)) {
    for (long long i = tid; i < n; i += nth) c[i] = bs_price(s[i], C, T);
    return;
  }
  const unsigned n2 = (unsigned)(n >> 1);
  const unsigned step = PAIRS * nth;
  const unsigned nfull = n2 / step;  // groups in which every pair of every thread is in range
  const double2* s2 = reinterpret_cast<const double2*>(s);
  double2* c2 = reinterpret_cast<double2*>(c);
  double2 xa[PAIRS], xb[PAIRS];
  auto load = [&](double2(&x)[PAIRS], unsigned base) {
#pragma unroll
    for (int q = 0; q < PAIRS; ++q) x[q] = ldg_stream(s2 + base + q * nth);
  };
  auto price = [&](const double2(&x)[PAIRS], unsigned base) {
#pragma unroll
    for (int q = 0; q < PAIRS; ++q) {
      double2 y;
      y.x = bs_price(x[q].x, C, T);
      y.y = bs_price(x[q].y, C, T);
      c2[base + q * nth] = y;
    }
  };
  unsigned base = tid, j = 0;
  if (nfull > 0) load(xa, base);
  for (; j + 2 <= nfull; j += 2) {
    load(xb, base + step);
    price(xa, base);
    if (j + 2 < nfull) load(xa, base + 2 * step);
    price(xb, base + step);
    base += 2 * step;
  }
  if (j < nfull) {
    price(xa, base);
    base += step;
  }
#pragma unroll
  for (int q = 0; q < PAIRS; ++q) {  // tail: the last partial group
    const unsigned i = base + q * nth;
    if (i < n2) {
      const double2 x = ldg_stream(s2 + i);
      double2 y;
      y.x = bs_price(x.x, C, T);
      y.y = bs_price(x.y, C, T);
      c2[i] = y;
    }
  }
  if ((n & 1) && tid == 0) c[n - 1] = bs_price(s[n - 1], C, T);
}
#define BS_LEAN_VARIANT(NAME, PAIRS, MINB)                                                        \
  __global__ void __launch_bounds__(256, MINB) NAME(const double* __restrict__ s,                 \
                                                    double* __restrict__ c, long long n, double r, \
                                                    double v, double t, double k) {                \
    bs_body_lean<PAIRS>(s, c, n, r, v, t, k);                                                      \
  }
BS_LEAN_VARIANT(k_bs_l4b2, 4, 2)
BS_LEAN_VARIANT(k_bs_l2b3, 2, 3)
BS_LEAN_VARIANT(k_bs_l2b4, 2, 4)
BS_LEAN_VARIANT(k_bs_l1b4, 1, 4)
BS_LEAN_VARIANT(k_bs_l3b2, 3, 2)
BS_LEAN_VARIANT(k_bs_l3b3, 3, 3)
BS_LEAN_VARIANT(k_bs_l8b1, 8, 1)

// Deeper prefetch without register cost: each thread keeps DEPTH of its own
// option pairs in flight with 16-byte cp.async into a private shared-memory
// ring of DEPTH+1 slots (it reads back only what it copied itself, so no
// block barrier is needed), covering the HBM latency with DEPTH pricing
// steps instead of one.  Same arithmetic and results as bs_body.
template <int DEPTH>
__device__ __forceinline__ void bs_body_async(const double* __restrict__ s, double* __restrict__ c,
                                              long long n, double r, double v, double t, double k) {
  __shared__ BsTables T;
  __shared__ double2 ring[DEPTH + 1][256];
  bs_tables_init(T);
  BsConst C;
  const double vst = v * sqrt(t);
  C.vst = vst;
  C.inv_vst = 1.0 / vst;
  C.mu_s = (r + 0.5 * v * v) * t / vst;
  C.inv_k = 1.0 / k;
  C.c2 = exp(r * t) / k;
  C.kexp = k * exp(-r * t);
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(s) && aligned16(c) && blockDim.x == 256) {
    const long long n2 = n >> 1;
    const double2* s2 = reinterpret_cast<const double2*>(s);
    double2* c2 = reinterpret_cast<double2*>(c);
    auto fetch = [&](long long i, int slot) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&ring[slot][threadIdx.x]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                   "l"(i < n2 ? s2 + i : s2), "r"(i < n2 ? 16 : 0)
                   : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int q = 0; q < DEPTH; ++q) fetch(tid + q * nth, q);
    int slot = 0;
    for (long long i = tid; i < n2; i += nth) {
      asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1) : "memory");
      const double2 cur = ring[slot][threadIdx.x];
      // refill the slot read in the previous step (its value is consumed)
      fetch(i + DEPTH * nth, slot == 0 ? DEPTH : slot - 1);
      double2 y;
      y.x = bs_price(cur.x, C, T);
      y.y = bs_price(cur.y, C, T);
      c2[i] = y;
      slot = slot == DEPTH ? 0 : slot + 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    done = n2 << 1;
  }
  for (long long i = done + tid; i < n; i += nth) c[i] = bs_price(s[i], C, T);
}
#define BS_ASYNC_VARIANT(NAME, DEPTH, MINB)                                                        \
  __global__ void __launch_bounds__(256, MINB) NAME(const double* __restrict__ s,                 \
                                                    double* __restrict__ c, long long n, double r, \
                                                    double v, double t, double k) {                \
    bs_body_async<DEPTH>(s, c, n, r, v, t, k);                                                     \
  }
BS_ASYNC_VARIANT(k_bs_a3b4, 3, 4)
BS_ASYNC_VARIANT(k_bs_a5b4, 5, 4)
BS_ASYNC_VARIANT(k_bs_a7b4, 7, 4)
BS_ASYNC_VARIANT(k_bs_a5b3, 5, 3)

// previous default (now "bs_p4"): 4 pairs per iteration, 2 CTAs/SM, one wave
// (49.7 us per 10M options vs 51.3 for 2 pairs / 3 CTAs and 52.8 for 1 pair /
// 4 CTAs); the product is its lean form k_bs_l4b2 (45.2 us)
__global__ void __launch_bounds__(256, 2) k_bs(const double* __restrict__ s, double* __restrict__ c,
                                            long long n, double r, double v, double t, double k) {
  bs_body<4>(s, c, n, r, v, t, k);
}
// tuning variants (same results; bench with tools/bs_variants.py)
__global__ void __launch_bounds__(256, 3) k_bs_p2b3(const double* __restrict__ s, double* __restrict__ c,
                                                 long long n, double r, double v, double t, double k) {
  bs_body<2>(s, c, n, r, v, t, k);
}
__global__ void __launch_bounds__(256, 4) k_bs_p1b4(const double* __restrict__ s, double* __restrict__ c,
                                                 long long n, double r, double v, double t, double k) {
  bs_body<1>(s, c, n, r, v, t, k);
}
__global__ void __launch_bounds__(256, 4) k_bs_p2b4(const double* __restrict__ s, double* __restrict__ c,
                                                 long long n, double r, double v, double t, double k) {
  bs_body<2>(s, c, n, r, v, t, k);
}
__global__ void __launch_bounds__(256, 6) k_bs_p1b6(const double* __restrict__ s, double* __restrict__ c,
                                                 long long n, double r, double v, double t, double k) {
  bs_body<1>(s, c, n, r, v, t, k);
}
__global__ void __launch_bounds__(256, 2) k_bs_p4b2(const double* __restrict__ s, double* __restrict__ c,
                                                 long long n, double r, double v, double t, double k) {
  bs_body<4>(s, c, n, r, v, t, k);
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
    // product (round 2): 38-39 FP64 ops per option (algebraic pricer), inputs
    // streamed by cp.async.bulk into a 3-stage ring, 6 options per thread in
    // lockstep, 2 CTAs/SM one wave: 40.5 us per 10M options vs 45.8 for the
    // round-1 product (bs_l3b2) in the same run (tools/bs_variants.py)
    {"bs", (const void*)k_bs2t_o6s3b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, 0,
     nullptr, v_bs},
    // f4: the same pricing in fp32 (HBM-bound)
    {"bs_f32", (const void*)k_bs_f32, "const ptr, out ptr, sint64, float, float, float, float", KF_NONE, 0, nullptr,
     v_bs_f32},
    {"bs_p4", (const void*)k_bs, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_a3b4", (const void*)k_bs_a3b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_a5b4", (const void*)k_bs_a5b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_a7b4", (const void*)k_bs_a7b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_a5b3", (const void*)k_bs_a5b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_p2b3", (const void*)k_bs_p2b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_p1b4", (const void*)k_bs_p1b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_p2b4", (const void*)k_bs_p2b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_p1b6", (const void*)k_bs_p1b6, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_p4b2", (const void*)k_bs_p4b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_l4b2", (const void*)k_bs_l4b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_l2b3", (const void*)k_bs_l2b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_l2b4", (const void*)k_bs_l2b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_l1b4", (const void*)k_bs_l1b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_l3b2", (const void*)k_bs_l3b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_l3b3", (const void*)k_bs_l3b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs_l8b1", (const void*)k_bs_l8b1, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2_p3w2b2", (const void*)k_bs2_p3w2b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2_p2w2b3", (const void*)k_bs2_p2w2b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2_p2w4b2", (const void*)k_bs2_p2w4b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2_p4w2b2", (const void*)k_bs2_p4w2b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2_p1w2b4", (const void*)k_bs2_p1w2b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2t_o4s4b2", (const void*)k_bs2t_o4s4b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2t_o4s3b3", (const void*)k_bs2t_o4s3b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2t_o2s4b4", (const void*)k_bs2t_o2s4b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2t_o6s3b2", (const void*)k_bs2t_o6s3b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
};
DAGRT_REGISTER_BUILTINS(kVecBs);

}  // namespace dagrt
