// Experimental B&S variants (libdagrt_exp.so; see exp_common.cuh): the
// round-1 kernels (46 FP64 ops per option: bs_p4, register / cp.async
// prefetch depths, lean loops), the round-2 lockstep pricer with register
// prefetch (bs2_*) and other TMA-ring shapes (bs2t_*).  Same results as the
// product within the fp64 tolerance; tested in tests/test_gpu_vec_bs.py.
#include "../bs_math.cuh"
#include "exp_common.cuh"

namespace dagrt {

// ---------------------------------------------------------------- B&S, round 2b
// The lean pricer with two FP64 instructions and ~4 integer instructions
// fewer per option (32 FP64 in the loop), tables from constant memory images:
//   * d1 is carried SCALED, ds = kappa d1 with kappa = sqrt(64 / ln 2), so
//     that -d1^2/2 = -ds^2 ln2/128: the exp's range reduction is
//     t = fma(-ds, ds, 1.5 2^52) (n = round(-ds^2) from the exact square),
//     rho = fma(ds, ds, n) -- the square is never formed on its own (3 FP64
//     instead of h, t, nd, r2); kappa is folded into every constant that
//     touches d1 (the log polynomial, the per-CTA table, d2's offset, the
//     A&S p);
//   * ln S: r = fma(S, inv[j] 2^-e, -1) with the 2^-e applied to the table
//     value's exponent field in place (no mantissa extraction, no register
//     copy), the polynomial pre-multiplied by kappa / (V sqrt T), and the
//     per-CTA table TL[j] = -ln(inv[j]) kappa / (V sqrt T) + kappa mu
//     interleaved with inv[j] (one 16-byte shared load per option):
//     ds = fma(e, kappa ln2 / (V sqrt T), fma(p, r, TL[j])) -- 5 FP64 from S to
//     ds instead of 6;
//   * inv / -ln inv / 2^(j/128) are exact hex images (bs_tables.inc,
//     tools/gen_bs_tables.py) copied into shared memory: no libdevice log /
//     exp2 per CTA (~2.5% of the kernel's FP64 work).
// Same formulas (SURVEY §8(c2) B&S: A&S 26.2.17, fp64), same truncation
// errors as the lean pricer (log series to r^3 with |r| <= 2^-10, exp series
// to rho^3 with |rho ln2/128| <= ln2/256).
#include "bs_tables.inc"

struct BsTabsM {
  double2 lt[512];  // {inv[j], TL[j]}
  double exp2j[128];
};
struct BsConstM {
  double c1, c2, c3;  // g, -g/2, g/3 with g = kappa / (V sqrt T): kappa x the log series
  double ln2g;        // ln2 g
  double vk;          // kappa V sqrt T (ds2 = ds1 - vk)
  double as;          // A&S p / kappa
  double nkexp;       // -K e^{-RT}
};
enum { kcMRound, kcMNegC3, kcMC2, kcMNegC, kcMCount };
static __constant__ double kBsM[kcMCount] = {
    6755399441055744.0,          // 1.5 2^52
    -2.6466421444330967e-08,     // -(ln2/128)^3 / 6
    1.4662262387640423e-05,      // (ln2/128)^2 / 2
    -0.0054152123481245725};     // -ln2/128
constexpr double kKappa = 9.608979270291599;  // sqrt(64 / ln 2)

// Per-CTA: constants and tables (TL depends on the launch's V, T, K, R).
__device__ __forceinline__ void bs_m_setup(BsTabsM& T, BsConstM& C, double r, double v, double t, double k) {
  const double vst = v * sqrt(t);
  const double ivst = 1.0 / vst;
  const double g = kKappa * ivst;
  const double mu_lnk = ((r + 0.5 * v * v) * t - log(k)) * ivst;  // d1 = ln S / (V sqrt T) + mu_lnk
  const double muk = kKappa * mu_lnk;
  C.c1 = g;
  C.c2 = -0.5 * g;
  C.c3 = g / 3.0;
  C.ln2g = 0.6931471805599453 * g;
  C.vk = kKappa * vst;
  C.as = kBsK[kcA] / kKappa;
  C.nkexp = -k * exp(-r * t);
  for (int j = threadIdx.x; j < 512; j += blockDim.x) {
    const double2 q = __ldg(reinterpret_cast<const double2*>(kBsLogTab) + j);  // {inv, -ln inv}
    T.lt[j] = make_double2(q.x, fma(q.y, g, muk));
    if (j < 128) T.exp2j[j] = __ldg(kBsExp2Tab + j);
  }
}

template <int W>
__device__ __forceinline__ void bs_price_m(const double (&s)[W], double (&out)[W], const BsConstM& C,
                                           const BsTabsM& T) {
  const double B1 = kBsK[kcB1], B2 = kBsK[kcB2], B3 = kBsK[kcB3], B4 = kBsK[kcB4], B5 = kBsK[kcB5];
  double d1[W], d2[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const int hi = __double2hiint(s[w]);
    const int eb = hi >> 20;                      // biased exponent (S positive)
    const double2 q = T.lt[(hi >> 11) & 511];     // {inv[j], TL[j]}
    // inv[j] 2^-(eb - 1023): the table value's exponent field lowered in place
    const double ie = __hiloint2double(__double2hiint(q.x) - ((eb - 1023) << 20), __double2loint(q.x));
    const double r = fma(s[w], ie, -1.0);         // = m inv[j] - 1, |r| <= 2^-10
    double p = fma(r, C.c3, C.c2);
    p = fma(r, p, C.c1);                           // g (1 - r/2 + r^2/3)
    d1[w] = fma((double)(eb - 1023), C.ln2g, fma(p, r, q.y));  // kappa d1
    d2[w] = d1[w] - C.vk;
  }
  double e1[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    // |ds| clamped to ~359 (ds^2 ln2/128 <= ~700: exp(-700) ~ 1e-304 stands
    // for 0 and the 2^(n/128) scaling stays in the normal range)
    const double dc = __hiloint2double(min(__double2hiint(d1[w]) & 0x7fffffff, 0x40767000), __double2loint(d1[w]));
    const double t = fma(-dc, dc, kBsM[kcMRound]);
    const int n = __double2loint(t);               // round(-ds^2)
    const double rho = fma(dc, dc, t - kBsM[kcMRound]);  // ds^2 + n, |rho| <= 1/2
    double p = fma(rho, kBsM[kcMNegC3], kBsM[kcMC2]);
    p = fma(rho, p, kBsM[kcMNegC]);
    p = fma(rho, p, 1.0);                          // e^{-rho ln2/128}
    const double sc = T.exp2j[n & 127] * p;
    e1[w] = __hiloint2double(__double2hiint(sc) + ((n >> 7) << 20), __double2loint(sc));  // e^{-d1^2/2}
  }
  double k1[W], k2[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const double D1 = fma(C.as, fabs(d1[w]), 1.0), D2 = fma(C.as, fabs(d2[w]), 1.0);
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
    const double k1s = __hiloint2double(__double2hiint(k1[w]) ^ (u1 ? 0x80000000 : 0), __double2loint(k1[w]));
    const double k2s = __hiloint2double(__double2hiint(k2[w]) ^ (u2 ? 0 : 0x80000000), __double2loint(k2[w]));
    const double m = fma(q1, k1s, q2 * k2s);
    const double u1d = __hiloint2double(u1 ? 0x3FF00000 : 0, 0);
    const double nk = __hiloint2double(u2 ? __double2hiint(C.nkexp) : 0, u2 ? __double2loint(C.nkexp) : 0);
    out[w] = fma(s[w], fma(e1[w], m, u1d), nk);
  }
}

// The TMA-staged body for the round-2b pricer: the ring's first bulk copies
// are issued BEFORE the per-CTA table setup, so the setup overlaps them.
template <int OPT, int STAGES>
__device__ __forceinline__ void bs2m_tma_body(const double* __restrict__ s, double* __restrict__ c, long long n,
                                              double r, double v, double t, double k) {
  constexpr int kChunk = 256 * OPT;
  __shared__ BsTabsM T;
  __shared__ __align__(128) double ring[STAGES][kChunk];
  __shared__ uint64_t full[STAGES];
  BsConstM C;
  const int tid = threadIdx.x;
  const bool fast = aligned16(s) && aligned16(c) && blockDim.x == 256;
  const long long nfullc = fast ? n / kChunk : 0;
  const long long G = gridDim.x;
  if (tid == 0) {
    for (int q = 0; q < STAGES; ++q) bs_mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < STAGES; ++q) {
      const long long ch = blockIdx.x + q * G;
      if (ch < nfullc) bs_bulk_g2s(ring[q], s + ch * kChunk, kChunk * 8, &full[q]);
    }
  }
  bs_m_setup(T, C, r, v, t, k);
  __syncthreads();  // tables and barrier initialisation visible
  int it = 0;
  for (long long ch = blockIdx.x; ch < nfullc; ch += G, ++it) {
    const int st = it % STAGES;
    bs_mbar_wait(&full[st], (unsigned)((it / STAGES) & 1));
    double a[OPT], o[OPT];
#pragma unroll
    for (int q = 0; q < OPT / 2; ++q) {
      const double2 x = reinterpret_cast<const double2*>(ring[st])[tid + 256 * q];
      a[2 * q] = x.x;
      a[2 * q + 1] = x.y;
    }
    __syncthreads();
    if (tid == 0 && ch + STAGES * G < nfullc) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bs_bulk_g2s(ring[st], s + (ch + STAGES * G) * kChunk, kChunk * 8, &full[st]);
    }
    bs_price_m<OPT>(a, o, C, T);
    double2* dst = reinterpret_cast<double2*>(c + ch * kChunk);
#pragma unroll
    for (int q = 0; q < OPT / 2; ++q) dst[tid + 256 * q] = make_double2(o[2 * q], o[2 * q + 1]);
  }
  const long long stride = G * blockDim.x;
  for (long long i = nfullc * kChunk + (long long)blockIdx.x * blockDim.x + tid; i < n; i += stride) {
    double a[1] = {s[i]}, o[1];
    bs_price_m<1>(a, o, C, T);
    c[i] = o[0];
  }
}

#define BS2M_VARIANT(NAME, OPT, STAGES, MINB)                                                      \
  __global__ void __launch_bounds__(256, MINB) NAME(const double* __restrict__ s,                 \
                                                    double* __restrict__ c, long long n, double r, \
                                                    double v, double t, double k) {                \
    bs2m_tma_body<OPT, STAGES>(s, c, n, r, v, t, k);                                               \
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

BS2T_VARIANT(k_bs2t_o4s4b2, 4, 4, 2)
BS2T_VARIANT(k_bs2t_o4s3b3, 4, 3, 3)
BS2T_VARIANT(k_bs2t_o2s4b4, 2, 4, 4)
BS2T_VARIANT(k_bs2t_o6s3b2, 6, 3, 2)  // the product shape, for side-by-side runs
BS2L_VARIANT(k_bs2l_o6s3b2, 6, 3, 2)
BS2L_VARIANT(k_bs2l_o4s3b3, 4, 3, 3)
BS2L_VARIANT(k_bs2l_o6s3b3, 6, 3, 3)
BS2L_VARIANT(k_bs2l_o6s2b3, 6, 2, 3)
BS2L_VARIANT(k_bs2l_o8s2b2, 8, 2, 2)
// Memory-path floor of the TMA-staged body: the same ring, loads, stores and
// table setup with the pricing replaced by one DMUL (tools/bs_variants.py).
struct BsPricerCopy {
  using Tables = BsTabsL;
  static __device__ __forceinline__ void init(Tables& T) { bs_tabsl_init(T); }
  template <int W>
  static __device__ __forceinline__ void price(const double (&s)[W], double (&o)[W], const BsConst& C,
                                               const Tables&) {
#pragma unroll
    for (int w = 0; w < W; ++w) o[w] = s[w] * C.inv_k;
  }
};
// compute-only form of the product (MODE 1: L2-resident input chunk, no stores)
__global__ void __launch_bounds__(256, 2) k_bs2x_o6s3b2(const double* __restrict__ s, double* __restrict__ c,
                                                        long long n, double r, double v, double t, double k) {
  bs2_tma_body<6, 3, BsPricerLean, 1>(s, c, n, r, v, t, k);
}
__global__ void __launch_bounds__(256, 2) k_bs2c_o6s3b2(const double* __restrict__ s, double* __restrict__ c,
                                                        long long n, double r, double v, double t, double k) {
  bs2_tma_body<6, 3, BsPricerCopy>(s, c, n, r, v, t, k);
}
// round-2b pricer (bs_price_m: 32 FP64 per option, constant tables, ring issued before the setup)
BS2M_VARIANT(k_bs2m_o6s3b2, 6, 3, 2)
BS2M_VARIANT(k_bs2m_o4s3b3, 4, 3, 3)
BS2M_VARIANT(k_bs2m_o6s3b3, 6, 3, 3)
BS2M_VARIANT(k_bs2m_o8s2b2, 8, 2, 2)
BS2M_VARIANT(k_bs2m_o4s4b2, 4, 4, 2)
BS3_VARIANT(k_bs3_o6s4b2, 6, 4, 2)
BS3_VARIANT(k_bs3_o6s6b2, 6, 6, 2)
BS3_VARIANT(k_bs3_o4s8b2, 4, 8, 2)
BS3_VARIANT(k_bs3_o4s6b3, 4, 6, 3)
BS3_VARIANT(k_bs3_o2s8b4, 2, 8, 4)
// warp-specialised ring with the lean (product) pricer: no CTA barrier per chunk
BS3L_VARIANT(k_bs3_o6s4b2l, 6, 4, 2)
BS3L_VARIANT(k_bs3_o6s6b2l, 6, 6, 2)
BS3L_VARIANT(k_bs3_o4s6b3l, 4, 6, 3)
BS3L_VARIANT(k_bs3_o4s8b2l, 4, 8, 2)

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

static const Builtin kBsExp[] = {
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
    // lean pricer (larger tables, one series term fewer each)
    {"bs2m_o6s3b2", (const void*)k_bs2m_o6s3b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2m_o4s3b3", (const void*)k_bs2m_o4s3b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2m_o6s3b3", (const void*)k_bs2m_o6s3b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2m_o8s2b2", (const void*)k_bs2m_o8s2b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2m_o4s4b2", (const void*)k_bs2m_o4s4b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2x_o6s3b2", (const void*)k_bs2x_o6s3b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2c_o6s3b2", (const void*)k_bs2c_o6s3b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2l_o6s3b2", (const void*)k_bs2l_o6s3b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2l_o4s3b3", (const void*)k_bs2l_o4s3b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2l_o6s3b3", (const void*)k_bs2l_o6s3b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2l_o6s2b3", (const void*)k_bs2l_o6s2b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    {"bs2l_o8s2b2", (const void*)k_bs2l_o8s2b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE},
    // warp-specialised (288 threads: 8 consumer warps + 1 producer warp)
    {"bs3_o6s4b2", (const void*)k_bs3_o6s4b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(6, 4)},
    {"bs3_o6s6b2", (const void*)k_bs3_o6s6b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(6, 6)},
    {"bs3_o4s8b2", (const void*)k_bs3_o4s8b2, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(4, 8)},
    {"bs3_o4s6b3", (const void*)k_bs3_o4s6b3, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(4, 6)},
    {"bs3_o6s4b2l", (const void*)k_bs3_o6s4b2l, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(6, 4)},
    {"bs3_o6s6b2l", (const void*)k_bs3_o6s6b2l, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(6, 6)},
    {"bs3_o4s6b3l", (const void*)k_bs3_o4s6b3l, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(4, 6)},
    {"bs3_o4s8b2l", (const void*)k_bs3_o4s8b2l, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(4, 8)},
    {"bs3_o2s8b4", (const void*)k_bs3_o2s8b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(2, 8)},
};
DAGRT_REGISTER_EXP(kBsExp);

}  // namespace dagrt
