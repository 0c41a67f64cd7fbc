// ML-ensemble kernels for sm_100a (§V-B; Fig. 6;
// Fig. 10; formulas: DESIGN.md reading R-ML).
//
// X is N x F int32 row-major (F = 200, L879-880), C = 10 classes.  Every
// kernel is HBM-bound; the row-wise ones use one thread per row (C floats =
// 40 B per row, 8-byte vector accesses, a warp covers 1280 contiguous bytes).
#include <type_traits>

#include "kcommon.cuh"

namespace dagrt {

constexpr int kMaxClasses = 16;

// mbarrier / bulk-copy helpers (NORM ring, MMUL tiles)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

// ---------------------------------------------------------------- NORM
// Z = (X - mu_f) / sd_f with population statistics, computed in ONE vertex:
// pass 1 exact integer column sums S = sum x (int64) and Q = sum x^2
// (unsigned 128-bit: exact for every int32 x and any N < 2^32) -> grid
// barrier -> one block per column reduces the per-block partials (integer,
// order-independent, so the statistics are bit-deterministic) and forms the
// variance from the exact integer N*Q - S^2 with ONE rounding -> grid barrier
// -> pass 2 normalises.  The kernel is registered cooperative: the scheduler
// launches it with cudaLaunchCooperativeKernel, which guarantees the whole
// grid is co-resident (the software barrier cannot deadlock against other
// vertices, another NORM in flight or an MPS SM limit).
//
// `stats` (out) layout: [0] u32 barrier, [1] u32 exit counter, pad to 16 B,
// then double mean[F], double inv_sd[F], then per block: int64 S[F],
// u64 Qlo[F], u64 Qhi[F]  (norm_stats_bytes(F, grid)).
struct NormHdr {
  unsigned bar;
  unsigned exitc;
  unsigned pad[2];
};
typedef unsigned __int128 u128;

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    volatile unsigned* vb = bar;
    while (*vb < target) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void acc_x(long long& s, u128& q, int v) {
  s += v;
  q += (unsigned long long)((long long)v * v);  // v^2 <= 2^62: exact in 64 bits
}

// u128 -> double: the two halves each round once (relative error < 2^-52)
__device__ __forceinline__ double u128_to_double(u128 v) {
  return (double)(unsigned long long)(v >> 64) * 18446744073709551616.0 +
         (double)(unsigned long long)v;
}

__global__ void __launch_bounds__(512, 2) k_norm(const int* __restrict__ X, float* __restrict__ Z,
                                              unsigned char* stats, long long N, int F) {
  extern __shared__ __align__(128) unsigned long long sh_u[];  // [RL][3F]: S, Qlo, Qhi per column (aliases the ring)
  NormHdr* hdr = reinterpret_cast<NormHdr*>(stats);
  double* mean = reinterpret_cast<double*>(stats + 16);
  double* inv = mean + F;
  unsigned long long* part = reinterpret_cast<unsigned long long*>(inv + F);  // [grid][3F]
  const int t = threadIdx.x;
  const bool vec = ((F & 3) == 0) && aligned16(X) && aligned16(Z) && (F / 4) <= 512;
  const int G = vec ? F / 4 : F;            // column groups (4 or 1 columns each)
  const int W = vec ? 4 : 1;
  const int RL = max(1, (int)blockDim.x / G); // row lanes
  const int g = t % G, rl = t / G;
  const bool active = rl < RL && G <= (int)blockDim.x;
  const long long rows_per = (N + gridDim.x - 1) / gridDim.x;
  const long long r0 = (long long)blockIdx.x * rows_per;
  const long long r1 = min(N, r0 + rows_per);

  // Ring path (vec, and dynamic shared memory for >= 2 chunks of CH = 2 RL
  // rows): the block's rows stream through shared memory by cp.async.bulk,
  // NST chunks in flight (one elected thread issues, an mbarrier per slot),
  // in pass 1 and again in pass 2 (whose first chunks are issued before the
  // grid barriers, so the statistics step overlaps them).  The register path
  // below had 4 x 16 B per thread in flight and was latency-bound (ncu:
  // long-scoreboard stalls dominate).  The per-thread partials' shared area
  // aliases the ring between the two passes.
  __shared__ uint64_t rfull[8];
  unsigned dyn;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  const int CH = 2 * RL;
  const unsigned slot_bytes = (unsigned)CH * (unsigned)F * 4u;
  const int NST = vec ? min(8, (int)(dyn / slot_bytes)) : 0;
  const bool ring = NST >= 2 && aligned16(X) && RL * G <= (int)blockDim.x;
  const long long nch = ring ? (r1 > r0 ? (r1 - r0) / CH : 0) : 0;  // whole chunks; the tail directly
  const int4* ringp = reinterpret_cast<const int4*>(sh_u);
  auto issue = [&](long long c, int st) {
    mbar_expect_tx(&rfull[st], slot_bytes);
    tma_bulk_g2s(reinterpret_cast<char*>(sh_u) + (size_t)st * slot_bytes, X + (r0 + c * CH) * F, slot_bytes,
                 &rfull[st]);
  };
  if (ring) {
    if (t == 0) {
      for (int st = 0; st < NST; ++st) mbar_init(&rfull[st], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int st = 0; st < NST && st < nch; ++st) issue(st, st);
    }
    __syncthreads();
  }
  unsigned it = 0;  // ring iterations (both passes): slot it % NST, parity (it / NST) & 1

  // ---- pass 1: exact column sums
  long long s[4] = {0, 0, 0, 0};
  u128 q[4] = {0, 0, 0, 0};
  if (ring) {
    for (long long c = 0; c < nch; ++c, ++it) {
      const int st = (int)(it % NST);
      mbar_wait(&rfull[st], (it / NST) & 1);
      int4 v[2] = {make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0)};
      if (active) {
        const int4* sl = ringp + (size_t)st * CH * G;
        v[0] = sl[rl * G + g];
        v[1] = sl[(rl + RL) * G + g];
      }
      __syncthreads();  // the slot is consumed: refill it
      if (t == 0 && c + NST < nch) issue(c + NST, st);
      if (active) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          acc_x(s[0], q[0], v[u].x); acc_x(s[1], q[1], v[u].y);
          acc_x(s[2], q[2], v[u].z); acc_x(s[3], q[3], v[u].w);
        }
      }
    }
    if (active) {
      const int4* X4 = reinterpret_cast<const int4*>(X);
      for (long long r = r0 + nch * CH + rl; r < r1; r += RL) {
        int4 v = ldg_stream(X4 + r * G + g);
        acc_x(s[0], q[0], v.x); acc_x(s[1], q[1], v.y);
        acc_x(s[2], q[2], v.z); acc_x(s[3], q[3], v.w);
      }
    }
  } else if (active) {
    if (vec) {
      const int4* X4 = reinterpret_cast<const int4*>(X);
      long long r = r0 + rl;
      for (; r + 3 * RL < r1; r += 4 * RL) {  // 4 independent 128-bit loads in flight
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ldg_stream(X4 + (r + u * RL) * G + g);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc_x(s[0], q[0], v[u].x); acc_x(s[1], q[1], v[u].y);
          acc_x(s[2], q[2], v[u].z); acc_x(s[3], q[3], v[u].w);
        }
      }
      for (; r < r1; r += RL) {
        int4 v = ldg_stream(X4 + r * G + g);
        acc_x(s[0], q[0], v.x); acc_x(s[1], q[1], v.y);
        acc_x(s[2], q[2], v.z); acc_x(s[3], q[3], v.w);
      }
    } else {
      for (long long r = r0 + rl; r < r1; r += RL) acc_x(s[0], q[0], X[r * F + g]);
    }
  }
  for (int w = 0; w < W; ++w) {
    if (active) {
      unsigned long long* row = sh_u + (size_t)rl * 3 * F;
      row[g * W + w] = (unsigned long long)s[w];
      row[F + g * W + w] = (unsigned long long)q[w];
      row[2 * F + g * W + w] = (unsigned long long)(q[w] >> 64);
    }
  }
  __syncthreads();
  for (int j = t; j < F; j += blockDim.x) {
    long long a = 0;
    u128 b = 0;
    for (int l = 0; l < RL; ++l) {
      const unsigned long long* row = sh_u + (size_t)l * 3 * F;
      a += (long long)row[j];
      b += ((u128)row[2 * F + j] << 64) | row[F + j];
    }
    unsigned long long* o = part + (size_t)blockIdx.x * 3 * F;
    o[j] = (unsigned long long)a;
    o[F + j] = (unsigned long long)b;
    o[2 * F + j] = (unsigned long long)(b >> 64);
  }
  const unsigned it2 = it;  // pass 2 starts at this ring iteration
  if (ring) {
    __syncthreads();  // the partials' reads of the (aliased) ring are done
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes before async-proxy writes
      for (int k = 0; k < NST && k < nch; ++k) issue(k, (int)((it2 + k) % NST));
    }
  }
  grid_barrier(&hdr->bar, gridDim.x);

  // ---- statistics: column j reduced by block j (and j + grid, ...), warp 0
  for (int j = blockIdx.x; j < F; j += gridDim.x) {
    if (t < 32) {
      long long a = 0;
      u128 b = 0;
      for (int k = t; k < (int)gridDim.x; k += 32) {
        const volatile unsigned long long* o = part + (size_t)k * 3 * F;
        a += (long long)o[j];
        b += ((u128)o[2 * F + j] << 64) | o[F + j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        const unsigned long long lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)b, o);
        const unsigned long long hi = __shfl_xor_sync(0xffffffffu, (unsigned long long)(b >> 64), o);
        b += ((u128)hi << 64) | lo;
      }
      if (t == 0) {
        // N^2 var = N Q - S^2, exact in 128 bits (N < 2^32), rounded once
        const __int128 S = a;
        const __int128 num = (__int128)((u128)N * b) - S * S;
        const double var = (num > 0 ? u128_to_double((u128)num) : 0.0) / ((double)N * (double)N);
        const double sd = sqrt(var);
        mean[j] = (double)a / (double)N;
        inv[j] = sd > 0.0 ? 1.0 / sd : 1.0;
      }
    }
  }
  grid_barrier(&hdr->bar, 2 * gridDim.x);

  // ---- pass 2: Z = (x - mu) * inv_sd
  if (ring) {
    float mu[4] = {0.f, 0.f, 0.f, 0.f}, is[4] = {0.f, 0.f, 0.f, 0.f};
    if (active)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        mu[w] = (float)((volatile double*)mean)[4 * g + w];
        is[w] = (float)((volatile double*)inv)[4 * g + w];
      }
    float4* Z4 = reinterpret_cast<float4*>(Z);
    it = it2;
    for (long long c = 0; c < nch; ++c, ++it) {
      const int st = (int)(it % NST);
      mbar_wait(&rfull[st], (it / NST) & 1);
      int4 v[2] = {make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0)};
      if (active) {
        const int4* sl = ringp + (size_t)st * CH * G;
        v[0] = sl[rl * G + g];
        v[1] = sl[(rl + RL) * G + g];
      }
      __syncthreads();
      if (t == 0 && c + NST < nch) issue(c + NST, st);
      if (active) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          float4 z;
          z.x = ((float)v[u].x - mu[0]) * is[0];
          z.y = ((float)v[u].y - mu[1]) * is[1];
          z.z = ((float)v[u].z - mu[2]) * is[2];
          z.w = ((float)v[u].w - mu[3]) * is[3];
          Z4[(r0 + c * CH + rl + u * RL) * G + g] = z;
        }
      }
    }
    if (active) {
      const int4* X4 = reinterpret_cast<const int4*>(X);
      for (long long r = r0 + nch * CH + rl; r < r1; r += RL) {
        int4 v = ldg_stream(X4 + r * G + g);
        float4 z;
        z.x = ((float)v.x - mu[0]) * is[0];
        z.y = ((float)v.y - mu[1]) * is[1];
        z.z = ((float)v.z - mu[2]) * is[2];
        z.w = ((float)v.w - mu[3]) * is[3];
        Z4[r * G + g] = z;
      }
    }
  } else if (active) {
    if (vec) {
      float mu[4], is[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        mu[w] = (float)((volatile double*)mean)[4 * g + w];
        is[w] = (float)((volatile double*)inv)[4 * g + w];
      }
      const int4* X4 = reinterpret_cast<const int4*>(X);
      float4* Z4 = reinterpret_cast<float4*>(Z);
      long long r = r0 + rl;
      for (; r + 3 * RL < r1; r += 4 * RL) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ldg_stream(X4 + (r + u * RL) * G + g);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float4 z;
          z.x = ((float)v[u].x - mu[0]) * is[0];
          z.y = ((float)v[u].y - mu[1]) * is[1];
          z.z = ((float)v[u].z - mu[2]) * is[2];
          z.w = ((float)v[u].w - mu[3]) * is[3];
          Z4[(r + u * RL) * G + g] = z;
        }
      }
      for (; r < r1; r += RL) {
        int4 v = ldg_stream(X4 + r * G + g);
        float4 z;
        z.x = ((float)v.x - mu[0]) * is[0];
        z.y = ((float)v.y - mu[1]) * is[1];
        z.z = ((float)v.z - mu[2]) * is[2];
        z.w = ((float)v.w - mu[3]) * is[3];
        Z4[r * G + g] = z;
      }
    } else {
      const float mu = (float)((volatile double*)mean)[g];
      const float is = (float)((volatile double*)inv)[g];
      for (long long r = r0 + rl; r < r1; r += RL) Z[r * F + g] = ((float)X[r * F + g] - mu) * is;
    }
  }
  // ---- reset the barrier for the next launch (last block out)
  __syncthreads();
  if (t == 0) {
    __threadfence();
    unsigned prev = atomicAdd(&hdr->exitc, 1u);
    if (prev == gridDim.x - 1) {
      hdr->bar = 0;
      hdr->exitc = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------- MMUL
// out[i, c] = sum_f A[i, f] W[c, f] (+ bias[c]); A int32 (NB, X) or fp32 (RR, Z).
// One thread per row; W (C x F fp32) staged in shared memory and read with
// broadcast 128-bit loads; A rows read with 128-bit loads.
template <typename T>
__device__ __forceinline__ float4 load4(const T* p);
template <>
__device__ __forceinline__ float4 load4<int>(const int* p) {
  int4 v = __ldg(reinterpret_cast<const int4*>(p));
  return make_float4((float)v.x, (float)v.y, (float)v.z, (float)v.w);
}
template <>
__device__ __forceinline__ float4 load4<float>(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

template <typename T, int C>
__device__ __forceinline__ void mmul_rows(const T* __restrict__ A, const float* __restrict__ sW,
                                          const float* __restrict__ bias, float* __restrict__ out,
                                          long long N, int F) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < N;
       r += (long long)gridDim.x * blockDim.x) {
    float acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = bias ? bias[c] : 0.f;
    const T* a = A + r * F;
    if ((F & 3) == 0 && aligned16(A)) {
      for (int f = 0; f < F; f += 4) {
        float4 x = load4<T>(a + f);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          float4 w = *reinterpret_cast<const float4*>(sW + c * F + f);
          acc[c] = fmaf(x.x, w.x, acc[c]);
          acc[c] = fmaf(x.y, w.y, acc[c]);
          acc[c] = fmaf(x.z, w.z, acc[c]);
          acc[c] = fmaf(x.w, w.w, acc[c]);
        }
      }
    } else {
      for (int f = 0; f < F; ++f) {
        float x = (float)a[f];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = fmaf(x, sW[c * F + f], acc[c]);
      }
    }
    float* o = out + r * C;
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = acc[c];
  }
}

template <typename T>
__device__ __forceinline__ void mmul_generic(const T* __restrict__ A, const float* __restrict__ sW,
                                             const float* __restrict__ bias, float* __restrict__ out,
                                             long long N, int F, int C) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < N;
       r += (long long)gridDim.x * blockDim.x) {
    for (int c = 0; c < C; ++c) {
      float acc = bias ? bias[c] : 0.f;
      for (int f = 0; f < F; ++f) acc = fmaf((float)A[r * F + f], sW[c * F + f], acc);
      out[r * C + c] = acc;
    }
  }
}

// TMA fast path (C = 10, F % 4 == 0, F <= 200, 128 threads): each CTA walks
// tiles of 64 consecutive rows.  A tile is ONE contiguous chunk of A
// (64 x 4F bytes), brought into shared memory by a single cp.async.bulk
// (TMA, completion on an mbarrier), double-buffered so the next tile streams
// in while this one is multiplied.  Two threads share a row (features
// [0, F/2) and [F/2, F)): with rows contiguous in smem their 128-bit reads
// are bank-conflict-free, the 10 weight rows are read with 2-address
// broadcast loads, and the two partial dot products are combined with one
// shuffle per class.  Per 4 features a warp issues 1 + 10 LDS.128 for 40 FFMA.
constexpr int kMmThreads = 128;
constexpr int kMmRows = kMmThreads / 2;  // rows per tile

template <typename T>
__device__ __forceinline__ float4 as_f4(const T* p);
template <>
__device__ __forceinline__ float4 as_f4<int>(const int* p) {
  const int4 v = *reinterpret_cast<const int4*>(p);
  return make_float4((float)v.x, (float)v.y, (float)v.z, (float)v.w);
}
template <>
__device__ __forceinline__ float4 as_f4<float>(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

// RPT = rows per thread: 1 (128 threads per 64-row tile, the round-2 form)
// or 2 (64 threads; thread pair k takes rows k and k + 32, so every weight
// load feeds 2 x 4 x 2 FMAs instead of 4 x 2 and the shared-memory wavefronts
// per FMA -- the kernel's bound, ncu -- drop to 28 / 80 from 24 / 40).
template <typename T, int RPT = 1>
__device__ __forceinline__ void mmul_tma10(const T* __restrict__ A, const float* __restrict__ sW,
                                           unsigned char* smem_tiles, uint64_t* full,
                                           const float* __restrict__ bias, float* __restrict__ out,
                                           long long N, int F) {
  const int t = threadIdx.x, h = t & 1, row = t >> 1;  // rows row, row + 32 (RPT 2)
  const int half = F / 2;                     // features per thread (multiple of 2)
  const size_t tile_bytes = (size_t)kMmRows * F * 4;
  auto buf = [&](int st) { return reinterpret_cast<T*>(smem_tiles + st * tile_bytes); };
  const long long ntiles = (N + kMmRows - 1) / kMmRows;
  float b[10];
#pragma unroll
  for (int c = 0; c < 10; ++c) b[c] = bias ? __ldg(bias + c) : 0.f;
  auto issue = [&](long long tile, int stage) {
    const long long r0 = tile * kMmRows;
    const unsigned bytes = (unsigned)(min((long long)kMmRows, N - r0) * F * 4);
    mbar_expect_tx(&full[stage], bytes);
    tma_bulk_g2s(buf(stage), A + r0 * F, bytes, &full[stage]);
  };
  if (t == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0) {
    if ((long long)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if ((long long)blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }
  int k = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int stage = k & 1;
    mbar_wait(&full[stage], (k >> 1) & 1);
    const long long r0 = tile * kMmRows;
    const int nrows = (int)min((long long)kMmRows, N - r0);
    float acc[RPT][10];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
      for (int c = 0; c < 10; ++c) acc[q][c] = h == 0 ? b[c] : 0.f;
    if (row < nrows) {  // (RPT 2: row + 32 may be past the tile's end; it then reads stale data, never stored)
      const T* xr = buf(stage) + (size_t)row * F + h * half;
      const float* wr = sW + h * half;
#pragma unroll 5
      for (int f = 0; f < half; f += 4) {
        float4 x[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) x[q] = as_f4<T>(xr + (size_t)q * 32 * F + f);
#pragma unroll
        for (int c = 0; c < 10; ++c) {
          const float4 w = *reinterpret_cast<const float4*>(wr + c * F + f);
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            acc[q][c] = fmaf(x[q].x, w.x, acc[q][c]);
            acc[q][c] = fmaf(x[q].y, w.y, acc[q][c]);
            acc[q][c] = fmaf(x[q].z, w.z, acc[q][c]);
            acc[q][c] = fmaf(x[q].w, w.w, acc[q][c]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
      for (int c = 0; c < 10; ++c) acc[q][c] += __shfl_xor_sync(0xffffffffu, acc[q][c], 1);
    if (RPT == 1) {
      if (row < nrows) {
        float2* o = reinterpret_cast<float2*>(out + (r0 + row) * 10);
        if (h == 0) {
          o[0] = make_float2(acc[0][0], acc[0][1]);
          o[1] = make_float2(acc[0][2], acc[0][3]);
        } else {
          o[2] = make_float2(acc[0][4], acc[0][5]);
          o[3] = make_float2(acc[0][6], acc[0][7]);
          o[4] = make_float2(acc[0][8], acc[0][9]);
        }
      }
    } else {  // lane h = 0 stores row `row`, lane h = 1 row `row + 32`
      const int rr = row + 32 * h;
      if (rr < nrows) {
        float2* o = reinterpret_cast<float2*>(out + (r0 + rr) * 10);
#pragma unroll
        for (int c = 0; c < 5; ++c)
          o[c] = h == 0 ? make_float2(acc[0][2 * c], acc[0][2 * c + 1])
                        : make_float2(acc[RPT - 1][2 * c], acc[RPT - 1][2 * c + 1]);
      }
    }
    __syncthreads();  // every thread is done with buf[stage]
    if (t == 0 && tile + 2 * (long long)gridDim.x < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile + 2 * (long long)gridDim.x, stage);
    }
  }
}

// shared-memory bytes of the TMA path: W, 2 mbarriers, two row tiles
__host__ __device__ constexpr size_t mmul_tma_smem(int F) {
  return (size_t)10 * F * 4 + 16 + 2 * (size_t)kMmRows * F * 4;
}

template <typename T>
__device__ __forceinline__ void mmul_body(const T* A, const float* W, const float* bias, float* out,
                                          long long N, int F, int C) {
  extern __shared__ __align__(16) float sW[];
  for (int i = threadIdx.x; i < C * F; i += blockDim.x) sW[i] = W[i];
  __syncthreads();
  const bool tma = C == 10 && (F & 3) == 0 && F <= 200 && ((F / 2) & 3) == 0 &&
                   (blockDim.x == kMmThreads || blockDim.x == kMmThreads / 2) && aligned16(A) &&
                   (((uintptr_t)out) & 7) == 0;
  if (tma) {
    uint64_t* full = reinterpret_cast<uint64_t*>(sW + 10 * F);   // 10F*4 is a multiple of 16
    unsigned char* tiles = reinterpret_cast<unsigned char*>(full + 2);
    if (blockDim.x == kMmThreads) mmul_tma10<T, 1>(A, sW, tiles, full, bias, out, N, F);
    else mmul_tma10<T, 2>(A, sW, tiles, full, bias, out, N, F);
  } else if (C == 10) {
    mmul_rows<T, 10>(A, sW, bias, out, N, F);
  } else {
    mmul_generic<T>(A, sW, bias, out, N, F, C);
  }
}

// NB MMUL: r1 = X theta^T + prior (prior is a const input).
__global__ void __launch_bounds__(256) k_nb_mmul(const int* __restrict__ X,
                                                 const float* __restrict__ theta,
                                                 const float* __restrict__ prior,
                                                 float* __restrict__ r1, long long N, int F, int C) {
  mmul_body<int>(X, theta, prior, r1, N, F, C);
}

// RR MMUL: r2 = Z W^T.
__global__ void __launch_bounds__(256) k_rr_mmul(const float* __restrict__ Zm,
                                                 const float* __restrict__ W,
                                                 float* __restrict__ r2, long long N, int F, int C) {
  mmul_body<float>(Zm, W, nullptr, r2, N, F, C);
}

// ---------------------------------------------------------------- row-wise (C columns)
// C = 10 fast path: a thread owns a PAIR of rows = 20 floats = 5 x 128-bit
// accesses (row pairs are 80 B, so 16-B aligned); per-row scalars move as
// float2/int2.  Other C: one thread per row, scalar accesses.
#define ROW_LOOP for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < N; \
                      r += (long long)gridDim.x * blockDim.x)
#define PAIR_LOOP for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N / 2; \
                       i += (long long)gridDim.x * blockDim.x)
#define TAIL_ROW if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0)

__device__ __forceinline__ void ld20(const float* base, long long i, float (&v)[20]) {
  const float4* p = reinterpret_cast<const float4*>(base) + i * 5;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const float4 q = p[k];
    v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
  }
}
__device__ __forceinline__ void st20(float* base, long long i, const float (&v)[20]) {
  float4* p = reinterpret_cast<float4*>(base) + i * 5;
#pragma unroll
  for (int k = 0; k < 5; ++k) p[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
}
__device__ __forceinline__ bool pair_ok(int C, const void* a, const void* b = nullptr) {
  return C == 10 && aligned16(a) && (b == nullptr || (((uintptr_t)b) & 7) == 0);
}

// MAX: m[i] = max_c r1[i, c]
__device__ __forceinline__ float rmax(const float* p, int C) {
  float v = p[0];
  for (int c = 1; c < C; ++c) v = fmaxf(v, p[c]);
  return v;
}
__global__ void __launch_bounds__(256) k_rowmax(const float* __restrict__ r1, float* __restrict__ m,
                                                long long N, int C) {
  if (pair_ok(C, r1, m)) {
    PAIR_LOOP {
      float v[20];
      ld20(r1, i, v);
      reinterpret_cast<float2*>(m)[i] = make_float2(rmax(v, 10), rmax(v + 10, 10));
    }
    TAIL_ROW m[N - 1] = rmax(r1 + (N - 1) * C, C);
    return;
  }
  ROW_LOOP m[r] = rmax(r1 + r * C, C);
}

// LSE: l[i] = m[i] + ln sum_c exp(r1[i,c] - m[i])
__device__ __forceinline__ float rlse(const float* p, float mm, int C) {
  float s = 0.f;
  for (int c = 0; c < C; ++c) s += expf(p[c] - mm);
  return mm + logf(s);
}
__global__ void __launch_bounds__(256) k_lse(const float* __restrict__ r1, const float* __restrict__ m,
                                             float* __restrict__ l, long long N, int C) {
  if (pair_ok(C, r1, m) && (((uintptr_t)l) & 7) == 0) {
    PAIR_LOOP {
      float v[20];
      ld20(r1, i, v);
      const float2 mm = reinterpret_cast<const float2*>(m)[i];
      reinterpret_cast<float2*>(l)[i] = make_float2(rlse(v, mm.x, 10), rlse(v + 10, mm.y, 10));
    }
    TAIL_ROW l[N - 1] = rlse(r1 + (N - 1) * C, m[N - 1], C);
    return;
  }
  ROW_LOOP l[r] = rlse(r1 + r * C, m[r], C);
}

// EXP and ADDV are elementwise over the flat N*C array (element e belongs
// to row e / C, class e % C), so they stream it with fully coalesced 128-bit
// accesses instead of per-row 80-byte strides.
#define FLAT4_LOOP for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; \
                        i += (long long)gridDim.x * blockDim.x)

// EXP: r1[i,c] = exp(r1[i,c] - l[i])   (in place)
__global__ void __launch_bounds__(256) k_exp_sub(float* __restrict__ r1, const float* __restrict__ l,
                                                 long long N, int C) {
  const long long total = N * C;
  const long long n4 = (C >= 4 && aligned16(r1)) ? total / 4 : 0;
  float4* p4 = reinterpret_cast<float4*>(r1);
  FLAT4_LOOP {
    float4 v = p4[i];
    const long long e = 4 * i, r = e / C;
    const int rem = (int)(e - r * C);  // 4 elements span at most 2 rows (C >= 4)
    const float la = __ldg(l + r);
    const float lb = rem + 3 >= C ? __ldg(l + r + 1) : la;
    v.x = expf(v.x - la);
    v.y = expf(v.y - (rem + 1 < C ? la : lb));
    v.z = expf(v.z - (rem + 2 < C ? la : lb));
    v.w = expf(v.w - (rem + 3 < C ? la : lb));
    p4[i] = v;
  }
  for (long long e = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    r1[e] = expf(r1[e] - l[e / C]);
}

// ADDV: r2[i,c] += b[c]   (in place)
__global__ void __launch_bounds__(256) k_addv(float* __restrict__ r2, const float* __restrict__ b,
                                              long long N, int C) {
  __shared__ float sb[2 * kMaxClasses + 4];
  const bool small = C <= kMaxClasses;
  if (small && threadIdx.x < 2 * C + 4) sb[threadIdx.x] = __ldg(b + (threadIdx.x % C));
  __syncthreads();
  const long long total = N * C;
  const long long n4 = (small && aligned16(r2)) ? total / 4 : 0;
  float4* p4 = reinterpret_cast<float4*>(r2);
  FLAT4_LOOP {
    float4 v = p4[i];
    const int c0 = (int)((4 * i) % C);  // sb[c0 + j] = b[(c0 + j) % C]
    v.x += sb[c0];
    v.y += sb[c0 + 1];
    v.z += sb[c0 + 2];
    v.w += sb[c0 + 3];
    p4[i] = v;
  }
  for (long long e = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    r2[e] += b[e % C];
}

// SOFTMAX: row softmax in place (max-shifted)
__device__ __forceinline__ void rsoftmax(float* v, int C) {
  float m = v[0];
  for (int c = 1; c < C; ++c) m = fmaxf(m, v[c]);
  float s = 0.f;
  for (int c = 0; c < C; ++c) { v[c] = expf(v[c] - m); s += v[c]; }
  const float is = 1.f / s;
  for (int c = 0; c < C; ++c) v[c] *= is;
}
__global__ void __launch_bounds__(256) k_softmax(float* __restrict__ x, long long N, int C) {
  if (pair_ok(C, x)) {
    PAIR_LOOP {
      float v[20];
      ld20(x, i, v);
      rsoftmax(v, 10);
      rsoftmax(v + 10, 10);
      st20(x, i, v);
    }
    TAIL_ROW {
      float v[kMaxClasses];
      for (int c = 0; c < C; ++c) v[c] = x[(N - 1) * C + c];
      rsoftmax(v, C);
      for (int c = 0; c < C; ++c) x[(N - 1) * C + c] = v[c];
    }
    return;
  }
  ROW_LOOP {
    float v[kMaxClasses];
    const int CC = min(C, kMaxClasses);
    float* p = x + r * C;
    for (int c = 0; c < CC; ++c) v[c] = p[c];
    rsoftmax(v, CC);
    for (int c = 0; c < CC; ++c) p[c] = v[c];
  }
}

// ARGMAX: r[i] = lowest c maximising r1[i,c] + r2[i,c]
__device__ __forceinline__ int rargmax(const float* a, const float* b, int C) {
  float best = a[0] + b[0];
  int bi = 0;
  for (int c = 1; c < C; ++c) {
    const float s = a[c] + b[c];
    if (s > best) { best = s; bi = c; }
  }
  return bi;
}
__global__ void __launch_bounds__(256) k_argmax(const float* __restrict__ r1,
                                                const float* __restrict__ r2, int* __restrict__ out,
                                                long long N, int C) {
  if (pair_ok(C, r1, out) && aligned16(r2)) {
    PAIR_LOOP {
      float a[20], b[20];
      ld20(r1, i, a);
      ld20(r2, i, b);
      reinterpret_cast<int2*>(out)[i] = make_int2(rargmax(a, b, 10), rargmax(a + 10, b + 10, 10));
    }
    TAIL_ROW out[N - 1] = rargmax(r1 + (N - 1) * C, r2 + (N - 1) * C, C);
    return;
  }
  ROW_LOOP out[r] = rargmax(r1 + r * C, r2 + r * C, C);
}

// launch contracts (dagrt_launch validates them; builtin.h LaunchCheck)
static const char* v_norm(const LaunchCheck& L) {  // X, Z, stats, N, F
  const int64_t N = L.i(3);
  const int F = L.i32(4);
  if (N < 0 || N >= (1ll << 32) || F < 1) return "need 0 <= N < 2^32 rows and F >= 1 features";
  const uint64_t nf = (uint64_t)N * F;
  if (!fits(L, 0, 4 * nf) || !fits(L, 1, 4 * nf)) return "X and Z need 4 N F bytes";
  if (!fits(L, 2, 16 + 16ull * F + 24ull * F * L.grid[0])) return "stats need 16 + 16 F + 24 F grid bytes";
  if (L.block[0] > 512 || L.block[0] % 32 || L.block[1] != 1 || L.block[2] != 1 || L.grid[1] != 1 || L.grid[2] != 1)
    return "1-D launch, block a multiple of 32 <= 512";
  const bool vec = (F % 4 == 0) && ((L.vals[0] | L.vals[1]) % 16 == 0) && F / 4 <= 512;
  const int G = vec ? F / 4 : F;
  if (G > (int)L.block[0]) return "block smaller than the feature groups";
  const int RL = (int)L.block[0] / G > 1 ? (int)L.block[0] / G : 1;
  if (L.smem < 24u * F * RL) return "dynamic shared memory below 24 F (block / groups) bytes";
  if (L.real) {  // the software grid barrier needs the whole grid co-resident
    static int per_sm = -1, sms = 0;
    static unsigned last_block = 0, last_smem = 0;
    if (per_sm < 0 || last_block != L.block[0] || last_smem != L.smem) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaFuncSetAttribute((const void*)k_norm, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_norm, (int)L.block[0], L.smem))
        per_sm = 0;
      cudaGetLastError();
      last_block = L.block[0];
      last_smem = L.smem;
    }
    if ((long long)L.grid[0] > (long long)per_sm * sms) return "grid larger than the co-resident CTAs (cooperative)";
  }
  return nullptr;
}
template <bool NB>
static const char* v_mmul(const LaunchCheck& L) {  // A, W, [prior,] out, N, F, C
  const int o = NB ? 1 : 0;
  const int64_t N = L.i(3 + o);
  const int F = L.i32(4 + o), C = L.i32(5 + o);
  if (N < 0 || F < 1 || C < 1) return "need N >= 0, F >= 1, C >= 1";
  if (!fits(L, 0, 4ull * N * F) || !fits(L, 1, 4ull * C * F) || !fits(L, 2 + o, 4ull * N * C))
    return "A (4 N F), weights (4 C F) or output (4 N C) too small";
  if (NB && !fits(L, 2, 4ull * C)) return "prior needs 4 C bytes";
  if (L.nthreads() > 256 || L.block[1] != 1 || L.block[2] != 1) return "1-D block of <= 256 threads";
  if (L.smem < 4u * C * F) return "dynamic shared memory below 4 C F bytes";
  const bool tma = C == 10 && F % 4 == 0 && F <= 200 && (F / 2) % 4 == 0 &&
                   (L.block[0] == kMmThreads || L.block[0] == kMmThreads / 2) &&
                   L.vals[0] % 16 == 0 && L.vals[2 + o] % 8 == 0;
  if (tma && L.smem < mmul_tma_smem(F)) return "TMA path needs mmul_tma_smem(F) bytes of shared memory";
  return nullptr;
}
// row-wise kernels over an N x C score array: (arrays..., N, C)
static const char* v_rows(const LaunchCheck& L, int na, const int* per_row_classes) {
  const int64_t N = L.i(na);
  const int C = L.i32(na + 1);
  if (N < 0 || C < 1 || C > kMaxClasses) return "need N >= 0 and 1 <= C <= 16";
  for (int a = 0; a < na; ++a)  // 1: N x C scores, 0: N per-row values, -1: checked by the caller
    if (per_row_classes[a] >= 0 && !fits(L, a, 4ull * N * (per_row_classes[a] ? C : 1)))
      return "an array is smaller than its N x C / N";
  return L.nthreads() <= 256 ? nullptr : "at most 256 threads per CTA";
}
static const char* v_rowmax(const LaunchCheck& L) { static const int k[] = {1, 0}; return v_rows(L, 2, k); }
static const char* v_lse(const LaunchCheck& L) { static const int k[] = {1, 0, 0}; return v_rows(L, 3, k); }
static const char* v_exp_sub(const LaunchCheck& L) { static const int k[] = {1, 0}; return v_rows(L, 2, k); }
static const char* v_addv(const LaunchCheck& L) {
  static const int k[] = {1, -1};
  if (const char* e = v_rows(L, 2, k)) return e;
  return fits(L, 1, 4ull * L.i32(3)) ? nullptr : "bias needs 4 C bytes";
}
static const char* v_softmax(const LaunchCheck& L) { static const int k[] = {1}; return v_rows(L, 1, k); }
static const char* v_argmax(const LaunchCheck& L) { static const int k[] = {1, 1, 0}; return v_rows(L, 3, k); }

static const Builtin kMl[] = {
    {"norm", (const void*)k_norm, "const ptr, out ptr, out ptr, sint64, sint32", KF_COOPERATIVE, 96 * 1024, nullptr, v_norm},
    {"nb_mmul", (const void*)k_nb_mmul,
     "const ptr, const ptr, const ptr, out ptr, sint64, sint32, sint32", KF_NONE, 120 * 1024, nullptr, v_mmul<true>},
    {"rr_mmul", (const void*)k_rr_mmul, "const ptr, const ptr, out ptr, sint64, sint32, sint32",
     KF_NONE, 120 * 1024, nullptr, v_mmul<false>},
    {"rowmax", (const void*)k_rowmax, "const ptr, out ptr, sint64, sint32", KF_NONE, 0, nullptr, v_rowmax},
    {"lse", (const void*)k_lse, "const ptr, const ptr, out ptr, sint64, sint32", KF_NONE, 0, nullptr, v_lse},
    {"exp_sub", (const void*)k_exp_sub, "ptr, const ptr, sint64, sint32", KF_NONE, 0, nullptr, v_exp_sub},
    {"addv", (const void*)k_addv, "ptr, const ptr, sint64, sint32", KF_NONE, 0, nullptr, v_addv},
    {"softmax", (const void*)k_softmax, "ptr, sint64, sint32", KF_NONE, 0, nullptr, v_softmax},
    {"argmax", (const void*)k_argmax, "const ptr, const ptr, out ptr, sint64, sint32", KF_NONE, 0, nullptr, v_argmax},
};
DAGRT_REGISTER_BUILTINS(kMl);

}  // namespace dagrt
