// Black & Scholes pricing arithmetic shared by the product kernel
// (kernels_vec_bs.cu) and its experimental variants (exp/bs_variants.cu).
// fp64 throughout; formulas: DESIGN.md reading R-BS.
#pragma once
#include "kcommon.cuh"

namespace dagrt {

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
static __constant__ double kBsK[kcCount] = {
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
  double mu_lnk;   // mu_s - ln(K) / (V sqrt T): d1 from ln S directly (lean pricer)
  double nkexp;    // -K e^{-RT}
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
static __constant__ double kBs2K[kc2Count] = {
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

// Lean pricer: the same formulas with larger tables so that both series
// lose a term: a 512-entry log table (|r| <= 2^-10: ln(1+r) to r^3, the
// dropped r^4/4 is < 2.3e-13 absolute) and a 128-entry exp table (|r2/2| <=
// ln2/256: e^{-r2/2} to r2^3, the dropped term < 2.2e-12 relative); ln S
// instead of ln(S/K) (ln K folded into the constant term of d1) and
// C = S (e1 m + u1) - K e^{-RT} u2 with the indicators as selected constants
// and the CND signs applied to k before one DFMA sums the two terms -- 34
// instead of 39 FP64 instructions per option in the main loop.  Tables: 9 KB of
// shared memory.
struct BsTabsL {
  double inv[512];
  double lninv[512];
  double exp2j[128];
};
__device__ __forceinline__ void bs_tabsl_init(BsTabsL& T) {
  for (int j = threadIdx.x; j < 512; j += blockDim.x) {
    const double c = 1.0 / (1.0 + (j + 0.5) / 512.0);
    T.inv[j] = c;
    T.lninv[j] = -log(c);
    if (j < 128) T.exp2j[j] = exp2(j / 128.0);
  }
  __syncthreads();
}
enum { kcL2Ln2_128, kcLNeg64Ln2, kcLE1, kcLE2, kcLE3, kcLE4, kcLCount };
static __constant__ double kBsL[kcLCount] = {
    0.010830424696249145,     // 2 ln2 / 128
    -92.33248261689366,       // -64 / ln2  (t = round(-h/2 * 128/ln2))
    // e^{-r2/2} = 1 - r2/2 + r2^2/8 - r2^3/48 (|r2| <= 2 ln2/256)
    -1.0 / 48.0, 1.0 / 8.0, -0.5, 1.0};
__device__ __forceinline__ double bs_log_l(double x, const BsTabsL& T) {
  const int hi = __double2hiint(x), lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const int j = (hi >> 11) & 511;
  const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, lo);
  const double r = fma(m, T.inv[j], -1.0);
  double p = fma(r, kBsK[kcThird], -0.5);
  p = fma(r, p, 1.0);
  return fma((double)e, kBsK[kcLn2], fma(p, r, T.lninv[j]));
}
template <int W>
__device__ __forceinline__ void bs_price_l(const double (&s)[W], double (&out)[W], const BsConst& C,
                                           const BsTabsL& T) {
  const double B1 = kBsK[kcB1], B2 = kBsK[kcB2], B3 = kBsK[kcB3], B4 = kBsK[kcB4], B5 = kBsK[kcB5],
               A = kBsK[kcA];
  double d1[W], d2[W], h[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    d1[w] = fma(bs_log_l(s[w], T), C.inv_vst, C.mu_lnk);  // ln(S/K) = ln S - ln K, folded into mu
    d2[w] = d1[w] - C.vst;
    h[w] = d1[w] * d1[w];
  }
  double e1[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const double hc = __hiloint2double(min(__double2hiint(h[w]), 0x4095E000), __double2loint(h[w]));
    const double t = fma(hc, kBsL[kcLNeg64Ln2], kRound);
    const int n = __double2loint(t);
    const double nd = t - kRound;
    const double r2 = fma(nd, kBsL[kcL2Ln2_128], hc);
    double p = fma(r2, kBsL[kcLE1], kBsL[kcLE2]);
    p = fma(r2, p, kBsL[kcLE3]);
    p = fma(r2, p, kBsL[kcLE4]);
    const double sc = T.exp2j[n & 127] * p;
    e1[w] = __hiloint2double(__double2hiint(sc) + ((n >> 7) << 20), __double2loint(sc));
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
    const bool u1 = __double2hiint(d1[w]) > 0, u2 = __double2hiint(d2[w]) > 0;
    // m = sigma1 q1 k1 - sigma2 q2 k2 with the signs on k (integer pipe) and
    // one DFMA for the sum: two FP64 instructions instead of three
    const double k1s = __hiloint2double(__double2hiint(k1[w]) ^ (u1 ? 0x80000000 : 0), __double2loint(k1[w]));
    const double k2s = __hiloint2double(__double2hiint(k2[w]) ^ (u2 ? 0 : 0x80000000), __double2loint(k2[w]));
    const double m = fma(q1, k1s, q2 * k2s);
    // C = S (e1 m + u1) - K e^{-RT} u2: the indicators as selected constants
    const double u1d = __hiloint2double(u1 ? 0x3FF00000 : 0, 0);
    const double nk = __hiloint2double(u2 ? __double2hiint(C.nkexp) : 0, u2 ? __double2loint(C.nkexp) : 0);
    out[w] = fma(s[w], fma(e1[w], m, u1d), nk);
  }
}

// pricer policies of the TMA-staged body: the round-2 pricer (product) or the lean one
struct BsPricerR2 {
  using Tables = BsTables;
  static __device__ __forceinline__ void init(Tables& T) { bs_tables_init(T); }
  template <int W>
  static __device__ __forceinline__ void price(const double (&s)[W], double (&o)[W], const BsConst& C,
                                               const Tables& T) {
    bs_price_w<W>(s, o, C, T);
  }
};
struct BsPricerLean {
  using Tables = BsTabsL;
  static __device__ __forceinline__ void init(Tables& T) { bs_tabsl_init(T); }
  template <int W>
  static __device__ __forceinline__ void price(const double (&s)[W], double (&o)[W], const BsConst& C,
                                               const Tables& T) {
    bs_price_l<W>(s, o, C, T);
  }
};

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

// MODE (labs only): 0 = the kernel; 1 = compute only (every bulk copy reads
// the CTA's first chunk -- L2-resident -- and nothing is stored unless a
// price is NaN); 2 = memory only is BsPricerCopy (exp)
template <int OPT, int STAGES, class PR = BsPricerR2, int MODE = 0>
__device__ __forceinline__ void bs2_tma_body(const double* __restrict__ s, double* __restrict__ c, long long n,
                                             double r, double v, double t, double k) {
  constexpr int kChunk = 256 * OPT;  // options per chunk (blockDim.x == 256)
  __shared__ typename PR::Tables T;
  __shared__ __align__(128) double ring[STAGES][kChunk];
  __shared__ uint64_t full[STAGES];
  PR::init(T);
  BsConst C;
  const double vst = v * sqrt(t);
  C.vst = vst;
  C.inv_vst = 1.0 / vst;
  C.mu_s = (r + 0.5 * v * v) * t / vst;
  C.inv_k = 1.0 / k;
  C.c2 = exp(r * t) / k;
  C.kexp = k * exp(-r * t);
  C.mu_lnk = C.mu_s - log(k) * C.inv_vst;
  C.nkexp = -C.kexp;
  const int tid = threadIdx.x;
  if (!(aligned16(s) && aligned16(c)) || blockDim.x != 256) {
    for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < n; i += (long long)gridDim.x * blockDim.x) {
      double a[2] = {s[i], 1.0}, o[2];
      PR::template price<2>(a, o, C, T);
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
      if (ch < nfullc) bs_bulk_g2s(ring[q], s + (MODE == 1 ? (long long)blockIdx.x : ch) * kChunk, kChunk * 8, &full[q]);
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
      bs_bulk_g2s(ring[st], s + (MODE == 1 ? (long long)blockIdx.x : ch + STAGES * G) * kChunk, kChunk * 8, &full[st]);
    }
    PR::template price<OPT>(a, o, C, T);
    double2* dst = reinterpret_cast<double2*>(c + ch * kChunk);
#pragma unroll
    for (int q = 0; q < OPT / 2; ++q)
      if (MODE == 0 || o[2 * q] != o[2 * q] || o[2 * q + 1] != o[2 * q + 1])
        dst[tid + 256 * q] = make_double2(o[2 * q], o[2 * q + 1]);
  }
  for (long long i = nfullc * kChunk + (long long)blockIdx.x * blockDim.x + tid; i < n; i += G * blockDim.x) {
    double a[2] = {s[i], 1.0}, o[2];
    PR::template price<2>(a, o, C, T);
    c[i] = o[0];
  }
}
// Warp-specialised form: warp 8 of a 288-thread CTA is a producer that keeps
// a deeper ring (STAGES chunks of 256 * OPT options) filled with bulk copies;
// the 8 consumer warps wait only on the stage they need (full barrier) and
// release it with one arrival per warp (empty barrier, count 8) as soon as
// their options are in registers -- no CTA-wide barrier per chunk, so warps
// drift apart and the FP64 pipe is fed while others wait on memory (the
// bs2t form lost ~40% of the pipe to chunk-synchronous waits: ncu fp64 pipe
// 60%, barrier + long-scoreboard stalls, profiles/r2_ncu_*).
__device__ __forceinline__ void bs_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

template <int OPT, int STAGES, class PR = BsPricerR2>
__device__ __forceinline__ void bs3_ws_body(const double* __restrict__ s, double* __restrict__ c, long long n,
                                            double r, double v, double t, double k) {
  constexpr int kCons = 256;            // consumer threads (warps 0-7); warp 8 produces
  constexpr int kChunk = kCons * OPT;   // options per chunk
  __shared__ typename PR::Tables T;
  extern __shared__ __align__(128) unsigned char bs3_dyn[];  // the ring: STAGES * kChunk * 8 bytes (dynamic)
  double(*ring)[kChunk] = reinterpret_cast<double(*)[kChunk]>(bs3_dyn);
  __shared__ uint64_t full[STAGES], empty[STAGES];
  PR::init(T);
  BsConst C;
  const double vst = v * sqrt(t);
  C.vst = vst;
  C.inv_vst = 1.0 / vst;
  C.mu_s = (r + 0.5 * v * v) * t / vst;
  C.inv_k = 1.0 / k;
  C.c2 = exp(r * t) / k;
  C.kexp = k * exp(-r * t);
  C.mu_lnk = C.mu_s - log(k) * C.inv_vst;
  C.nkexp = -C.kexp;
  const int tid = threadIdx.x, warp = tid >> 5;
  unsigned dyn;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  if (!(aligned16(s) && aligned16(c)) || blockDim.x != kCons + 32 || dyn < STAGES * kChunk * 8u) {
    for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < n; i += (long long)gridDim.x * blockDim.x) {
      double a[2] = {s[i], 1.0}, o[2];
      PR::template price<2>(a, o, C, T);
      c[i] = o[0];
    }
    return;
  }
  const long long nfullc = n / kChunk;
  const long long G = gridDim.x;
  if (tid == 0) {
    for (int q = 0; q < STAGES; ++q) {
      bs_mbar_init(&full[q], 1);
      bs_mbar_init(&empty[q], kCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kCons / 32) {  // producer (one lane)
    if ((tid & 31) == 0) {
      int it = 0;
      for (long long ch = blockIdx.x; ch < nfullc; ch += G, ++it) {
        const int st = it % STAGES;
        if (it >= STAGES) bs_mbar_wait(&empty[st], (unsigned)((it / STAGES - 1) & 1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bs_bulk_g2s(ring[st], s + ch * kChunk, kChunk * 8, &full[st]);
      }
    }
    return;  // no CTA-wide barrier below this point
  }
  int it = 0;
  for (long long ch = blockIdx.x; ch < nfullc; ch += G, ++it) {
    const int st = it % STAGES;
    bs_mbar_wait(&full[st], (unsigned)((it / STAGES) & 1));
    double a[OPT], o[OPT];
#pragma unroll
    for (int q = 0; q < OPT / 2; ++q) {
      const double2 x = reinterpret_cast<const double2*>(ring[st])[tid + kCons * q];
      a[2 * q] = x.x;
      a[2 * q + 1] = x.y;
    }
    __syncwarp();
    if ((tid & 31) == 0) bs_mbar_arrive(&empty[st]);
    PR::template price<OPT>(a, o, C, T);
    double2* dst = reinterpret_cast<double2*>(c + ch * kChunk);
#pragma unroll
    for (int q = 0; q < OPT / 2; ++q) dst[tid + kCons * q] = make_double2(o[2 * q], o[2 * q + 1]);
  }
  for (long long i = nfullc * kChunk + (long long)blockIdx.x * kCons + tid; i < n; i += G * kCons) {
    double a[2] = {s[i], 1.0}, o[2];
    PR::template price<2>(a, o, C, T);
    c[i] = o[0];
  }
}
// dynamic shared memory of a bs3 instance (its ring)
#define BS3_SMEM(OPT, STAGES) ((STAGES) * 256 * (OPT) * 8)
#define BS3L_VARIANT(NAME, OPT, STAGES, MINB)                                                     \
  __global__ void __launch_bounds__(288, MINB) NAME(const double* __restrict__ s,                \
                                                    double* __restrict__ c, long long n, double r, \
                                                    double v, double t, double k) {                \
    bs3_ws_body<OPT, STAGES, BsPricerLean>(s, c, n, r, v, t, k);                                   \
  }
#define BS3_VARIANT(NAME, OPT, STAGES, MINB)                                                      \
  __global__ void __launch_bounds__(288, MINB) NAME(const double* __restrict__ s,                \
                                                    double* __restrict__ c, long long n, double r, \
                                                    double v, double t, double k) {                \
    bs3_ws_body<OPT, STAGES>(s, c, n, r, v, t, k);                                                 \
  }

#define BS2L_VARIANT(NAME, OPT, STAGES, MINB)                                                      \
  __global__ void __launch_bounds__(256, MINB) NAME(const double* __restrict__ s,                 \
                                                    double* __restrict__ c, long long n, double r, \
                                                    double v, double t, double k) {                \
    bs2_tma_body<OPT, STAGES, BsPricerLean>(s, c, n, r, v, t, k);                                  \
  }
#define BS2T_VARIANT(NAME, OPT, STAGES, MINB)                                                      \
  __global__ void __launch_bounds__(256, MINB) NAME(const double* __restrict__ s,                 \
                                                    double* __restrict__ c, long long n, double r, \
                                                    double v, double t, double k) {                \
    bs2_tma_body<OPT, STAGES>(s, c, n, r, v, t, k);                                                \
  }

}  // namespace dagrt
