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

// ---------------------------------------------------------------- NORM
// Z = (X - mu_f) / sd_f with population statistics, computed in ONE vertex:
// pass 1 exact integer column sums of x and x^2 -> grid barrier -> one block
// per column reduces the per-block partials (int64, order-independent, so the
// statistics are bit-deterministic) -> grid barrier -> pass 2 normalises.
// The grid (2 CTAs/SM x 148, 512 threads) is co-resident on an idle or
// shared B200 (the scheduler may run other vertices beside it; they do not
// wait on NORM, so its CTAs always become resident).
//
// `stats` (out) layout: [0] u32 barrier, [1] u32 exit counter, pad to 16 B,
// then double mean[F], double inv_sd[F], then int64 part[grid][2F].
struct NormHdr {
  unsigned bar;
  unsigned exitc;
  unsigned pad[2];
};

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

__global__ void __launch_bounds__(512) k_norm(const int* __restrict__ X, float* __restrict__ Z,
                                              unsigned char* stats, long long N, int F) {
  extern __shared__ long long sh_ll[];  // [RL][2F]
  NormHdr* hdr = reinterpret_cast<NormHdr*>(stats);
  double* mean = reinterpret_cast<double*>(stats + 16);
  double* inv = mean + F;
  long long* part = reinterpret_cast<long long*>(inv + F);
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

  // ---- pass 1: exact column sums (int32 per thread: <= 9*rows, 81*rows)
  int s[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
  if (active) {
    if (vec) {
      const int4* X4 = reinterpret_cast<const int4*>(X);
      for (long long r = r0 + rl; r < r1; r += RL) {
        int4 v = ldg_stream(X4 + r * G + g);
        s[0] += v.x; s[1] += v.y; s[2] += v.z; s[3] += v.w;
        q[0] += v.x * v.x; q[1] += v.y * v.y; q[2] += v.z * v.z; q[3] += v.w * v.w;
      }
    } else {
      for (long long r = r0 + rl; r < r1; r += RL) {
        int v = X[r * F + g];
        s[0] += v;
        q[0] += v * v;
      }
    }
  }
  for (int w = 0; w < W; ++w) {
    if (active) {
      sh_ll[(size_t)rl * 2 * F + g * W + w] = s[w];
      sh_ll[(size_t)rl * 2 * F + F + g * W + w] = q[w];
    }
  }
  __syncthreads();
  for (int j = t; j < 2 * F; j += blockDim.x) {
    long long a = 0;
    for (int l = 0; l < RL; ++l) a += sh_ll[(size_t)l * 2 * F + j];
    part[(size_t)blockIdx.x * 2 * F + j] = a;
  }
  grid_barrier(&hdr->bar, gridDim.x);

  // ---- statistics: column j reduced by block j (and j + grid, ...)
  __shared__ long long red[2][32];
  for (int j = blockIdx.x; j < F; j += gridDim.x) {
    long long a = 0, b = 0;
    for (int k = t; k < (int)gridDim.x; k += blockDim.x) {
      a += part[(size_t)k * 2 * F + j];
      b += part[(size_t)k * 2 * F + F + j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((t & 31) == 0) { red[0][t >> 5] = a; red[1][t >> 5] = b; }
    __syncthreads();
    if (t == 0) {
      long long S = 0, Q = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { S += red[0][w]; Q += red[1][w]; }
      const double mu = (double)S / (double)N;
      const double var = (double)Q / (double)N - mu * mu;
      const double sd = var > 0.0 ? sqrt(var) : 0.0;
      mean[j] = mu;
      inv[j] = sd > 0.0 ? 1.0 / sd : 1.0;
    }
    __syncthreads();
  }
  grid_barrier(&hdr->bar, 2 * gridDim.x);

  // ---- pass 2: Z = (x - mu) * inv_sd
  if (active) {
    if (vec) {
      float mu[4], is[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        mu[w] = (float)((volatile double*)mean)[4 * g + w];
        is[w] = (float)((volatile double*)inv)[4 * g + w];
      }
      const int4* X4 = reinterpret_cast<const int4*>(X);
      float4* Z4 = reinterpret_cast<float4*>(Z);
      for (long long r = r0 + rl; r < r1; r += RL) {
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

// Tiled fast path (C = 10, F % 40 == 0, 128 threads): a CTA takes tiles of
// 256 rows; the tile's X is staged through shared memory in 40-feature
// chunks with coalesced 128-bit loads (row stride padded to 44 words so the
// per-thread 128-bit reads are conflict-free); each thread accumulates TWO
// rows x 10 classes (the broadcast weight loads are reused for both rows):
// per 4 features 2 + 10 LDS.128 feed 80 FFMA, so the kernel is FFMA-bound
// below the HBM time instead of L1-bound on strided row reads.
constexpr int kMmThreads = 128;
constexpr int kMmRows = 2 * kMmThreads;
constexpr int kMmChunk = 40;
constexpr int kMmStride = kMmChunk + 4;
constexpr int kMmSmem = 4 * (10 * 200 + kMmRows * kMmStride);  // bytes for F = 200

template <typename T>
__device__ __forceinline__ float4 to_f4(const T& v);
template <>
__device__ __forceinline__ float4 to_f4<int4>(const int4& v) {
  return make_float4((float)v.x, (float)v.y, (float)v.z, (float)v.w);
}
template <>
__device__ __forceinline__ float4 to_f4<float4>(const float4& v) { return v; }

template <typename T, typename V4>
__device__ __forceinline__ void mmul_tiled10(const T* __restrict__ A, const float* __restrict__ sW,
                                             V4* __restrict__ sx, const float* __restrict__ bias,
                                             float* __restrict__ out, long long N, int F) {
  const int t = threadIdx.x;
  const int F4 = F / 4;
  const long long ntiles = (N + kMmRows - 1) / kMmRows;
  const V4* A4 = reinterpret_cast<const V4*>(A);
  float b[10];
#pragma unroll
  for (int c = 0; c < 10; ++c) b[c] = bias ? __ldg(bias + c) : 0.f;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long r0 = tile * kMmRows;
    const int nrows = (int)min((long long)kMmRows, N - r0);
    float a0[10], a1[10];
#pragma unroll
    for (int c = 0; c < 10; ++c) { a0[c] = b[c]; a1[c] = b[c]; }
    for (int f0 = 0; f0 < F; f0 += kMmChunk) {
      __syncthreads();  // the previous chunk has been consumed
      constexpr int G = kMmChunk / 4;  // 10 vectors per row chunk
#pragma unroll 4
      for (int k = t; k < kMmRows * G; k += kMmThreads) {
        const int rr = k / G, gg = k - rr * G;
        V4 v;
        if (rr < nrows) v = ldg_stream(A4 + (r0 + rr) * F4 + f0 / 4 + gg);
        else v = V4{0, 0, 0, 0};
        sx[rr * (kMmStride / 4) + gg] = v;
      }
      __syncthreads();
      const V4* x0p = sx + t * (kMmStride / 4);
      const V4* x1p = sx + (t + kMmThreads) * (kMmStride / 4);
#pragma unroll 2
      for (int g = 0; g < G; ++g) {
        const float4 x0 = to_f4(x0p[g]), x1 = to_f4(x1p[g]);
#pragma unroll
        for (int c = 0; c < 10; ++c) {
          const float4 w = *reinterpret_cast<const float4*>(sW + c * F + f0 + 4 * g);
          a0[c] = fmaf(x0.x, w.x, a0[c]);
          a0[c] = fmaf(x0.y, w.y, a0[c]);
          a0[c] = fmaf(x0.z, w.z, a0[c]);
          a0[c] = fmaf(x0.w, w.w, a0[c]);
          a1[c] = fmaf(x1.x, w.x, a1[c]);
          a1[c] = fmaf(x1.y, w.y, a1[c]);
          a1[c] = fmaf(x1.z, w.z, a1[c]);
          a1[c] = fmaf(x1.w, w.w, a1[c]);
        }
      }
    }
    if (t < nrows) {
      float2* o = reinterpret_cast<float2*>(out + (r0 + t) * 10);
#pragma unroll
      for (int c = 0; c < 5; ++c) o[c] = make_float2(a0[2 * c], a0[2 * c + 1]);
    }
    if (t + kMmThreads < nrows) {
      float2* o = reinterpret_cast<float2*>(out + (r0 + t + kMmThreads) * 10);
#pragma unroll
      for (int c = 0; c < 5; ++c) o[c] = make_float2(a1[2 * c], a1[2 * c + 1]);
    }
  }
}

template <typename T>
__device__ __forceinline__ void mmul_body(const T* A, const float* W, const float* bias, float* out,
                                          long long N, int F, int C) {
  extern __shared__ __align__(16) float sW[];
  for (int i = threadIdx.x; i < C * F; i += blockDim.x) sW[i] = W[i];
  __syncthreads();
  const bool tiled = C == 10 && F % kMmChunk == 0 && F <= 200 && blockDim.x == kMmThreads &&
                     aligned16(A) && (((uintptr_t)out) & 7) == 0;
  if (tiled) {
    using V4 = typename std::conditional<std::is_same<T, int>::value, int4, float4>::type;
    V4* sx = reinterpret_cast<V4*>(sW + 10 * F + ((10 * F) & 3 ? 4 - ((10 * F) & 3) : 0));
    mmul_tiled10<T, V4>(A, sW, sx, bias, out, N, F);
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

// EXP: r1[i,c] = exp(r1[i,c] - l[i])   (in place)
__global__ void __launch_bounds__(256) k_exp_sub(float* __restrict__ r1, const float* __restrict__ l,
                                                 long long N, int C) {
  if (pair_ok(C, r1, l)) {
    PAIR_LOOP {
      float v[20];
      ld20(r1, i, v);
      const float2 ll = reinterpret_cast<const float2*>(l)[i];
#pragma unroll
      for (int c = 0; c < 10; ++c) { v[c] = expf(v[c] - ll.x); v[10 + c] = expf(v[10 + c] - ll.y); }
      st20(r1, i, v);
    }
    TAIL_ROW for (int c = 0; c < C; ++c) r1[(N - 1) * C + c] = expf(r1[(N - 1) * C + c] - l[N - 1]);
    return;
  }
  ROW_LOOP {
    float* p = r1 + r * C;
    const float ll = l[r];
    for (int c = 0; c < C; ++c) p[c] = expf(p[c] - ll);
  }
}

// ADDV: r2[i,c] += b[c]   (in place)
__global__ void __launch_bounds__(256) k_addv(float* __restrict__ r2, const float* __restrict__ b,
                                              long long N, int C) {
  if (pair_ok(C, r2)) {
    float bb[10];
#pragma unroll
    for (int c = 0; c < 10; ++c) bb[c] = __ldg(b + c);
    PAIR_LOOP {
      float v[20];
      ld20(r2, i, v);
#pragma unroll
      for (int c = 0; c < 10; ++c) { v[c] += bb[c]; v[10 + c] += bb[c]; }
      st20(r2, i, v);
    }
    TAIL_ROW for (int c = 0; c < C; ++c) r2[(N - 1) * C + c] += b[c];
    return;
  }
  ROW_LOOP {
    float* p = r2 + r * C;
    for (int c = 0; c < C; ++c) p[c] += b[c];
  }
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

static const Builtin kMl[] = {
    {"norm", (const void*)k_norm, "const ptr, out ptr, out ptr, sint64, sint32", KF_NONE},
    {"nb_mmul", (const void*)k_nb_mmul,
     "const ptr, const ptr, const ptr, out ptr, sint64, sint32, sint32", KF_NONE, 96 * 1024},
    {"rr_mmul", (const void*)k_rr_mmul, "const ptr, const ptr, out ptr, sint64, sint32, sint32",
     KF_NONE, 96 * 1024},
    {"rowmax", (const void*)k_rowmax, "const ptr, out ptr, sint64, sint32", KF_NONE},
    {"lse", (const void*)k_lse, "const ptr, const ptr, out ptr, sint64, sint32", KF_NONE},
    {"exp_sub", (const void*)k_exp_sub, "ptr, const ptr, sint64, sint32", KF_NONE},
    {"addv", (const void*)k_addv, "ptr, const ptr, sint64, sint32", KF_NONE},
    {"softmax", (const void*)k_softmax, "ptr, sint64, sint32", KF_NONE},
    {"argmax", (const void*)k_argmax, "const ptr, const ptr, out ptr, sint64, sint32", KF_NONE},
};
DAGRT_REGISTER_BUILTINS(kMl);

}  // namespace dagrt
