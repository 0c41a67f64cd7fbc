// Experimental B&S variants (libdagrt_exp.so; see exp_common.cuh): the
// round-1 kernels (46 FP64 ops per option: bs_p4, register / cp.async
// prefetch depths, lean loops), the round-2 lockstep pricer with register
// prefetch (bs2_*) and other TMA-ring shapes (bs2t_*).  Same results as the
// product within the fp64 tolerance; tested in tests/test_gpu_vec_bs.py.
#include "../bs_math.cuh"
#include "exp_common.cuh"

namespace dagrt {

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
    {"bs3_o2s8b4", (const void*)k_bs3_o2s8b4, "const ptr, out ptr, sint64, double, double, double, double", KF_NONE, BS3_SMEM(2, 8)},
};
DAGRT_REGISTER_EXP(kBsExp);

}  // namespace dagrt
