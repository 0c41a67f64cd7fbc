// Kernels the scheduler itself launches (not benchmark vertices).
#include <cstdint>

#include "builtin.h"

namespace dagrt {

// Small host read (the host accesses an array and waits
// only for its producers): copy n bytes from device memory into MAPPED pinned
// host memory, make them visible to the host (__threadfence_system), then
// publish `seq` in the flag word the host spins on.  One CTA; reads of at
// most a few KB (the sink elements of resident mode, reduction scalars).
// Measured on the B200 box: kernel + host spin returns ~5 us sooner than a
// 4-byte cudaMemcpyAsync D2H + cudaStreamSynchronize (tools/launch_cost.cu).
__global__ void __launch_bounds__(256) k_read_mapped(const unsigned char* __restrict__ src,
                                                     unsigned char* dst, uint32_t n,
                                                     uint32_t* flag, uint32_t seq) {
  if ((((uintptr_t)src | (uintptr_t)dst | n) & 3u) == 0) {
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
    volatile uint32_t* d4 = reinterpret_cast<volatile uint32_t*>(dst);
    for (uint32_t i = threadIdx.x; i < n / 4; i += blockDim.x) d4[i] = s4[i];
  } else {
    volatile unsigned char* d = dst;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) d[i] = src[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t*>(flag) = seq;
}

const void* read_mapped_kernel() { return (const void*)k_read_mapped; }

}  // namespace dagrt

namespace dagrt {

// Peak probes (tools/box_peaks.py, SURVEY §8(d) "peaks to measure once per
// box"): `iters` x 8 independent FMA chains per thread, result kept live
// through a data-dependent store.  Not DAG vertices of any benchmark.
__global__ void __launch_bounds__(256) k_peak_dfma(double* out, long long iters) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  const double m = 1.0000001, c = 1e-7;
  for (long long k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, c);
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == -1.0) out[threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) k_peak_ffma(float* out, long long iters) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9f + i;
  const float m = 1.0000001f, c = 1e-7f;
  for (long long k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], m, c);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == -1.f) out[threadIdx.x] = s;
}

// Utility vertex: a[i] = alpha * a[i] + beta (in place, fp32).  Used by the
// scheduler tests (chains of dependent writes on one array) and as a cheap
// device-side initialiser; not a vertex of any benchmark DAG.
__global__ void __launch_bounds__(256) k_axpb(float* a, long long n, float alpha, float beta) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = fmaf(alpha, a[i], beta);
}

static const char* v_axpb(const LaunchCheck& L) {
  return fits(L, 0, 4ull * L.i(1)) ? nullptr : "a needs 4 n bytes";
}

static const Builtin kProbes[] = {
    {"axpb", (const void*)k_axpb, "ptr, sint64, float, float", KF_NONE, 0, nullptr, v_axpb},
    {"peak_dfma", (const void*)k_peak_dfma, "out ptr, sint64", KF_NONE},
    {"peak_ffma", (const void*)k_peak_ffma, "out ptr, sint64", KF_NONE},
};
DAGRT_REGISTER_BUILTINS(kProbes);

}  // namespace dagrt
