// Does integer work issue alongside the FP64 pipe? (tools only)
// Each thread runs 8 independent DFMA chains for `iters` iterations, plus
// INT independent integer ops per DFMA group (0, 8, 16, 32), at 16 warps per
// SM (2 CTAs x 256 threads x 148 SMs).  If the integer ops are free, time
// stays at the DFMA-only time; if every FP64 warp-instruction holds the
// dispatch port for 2 cycles, time grows by INT cycles per iteration per warp
// slot.  Result: ns per kernel -> cycles per DFMA warp-instruction per SMSP.
#include <cuda_runtime.h>
#include <stdint.h>

template <int INT>
__global__ void __launch_bounds__(256, 2) k_lab(double* out, int iters, unsigned seed) {
  double a[8];
  unsigned u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
    u[i] = seed + threadIdx.x * 7 + i;
  }
  const double m = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, c);
#pragma unroll
    for (int j = 0; j < INT; ++j) u[j & 7] = (u[j & 7] * 1664525u) ^ (u[(j + 3) & 7] >> 3);
  }
  double s = 0;
  unsigned t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    s += a[i];
    t ^= u[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (double)t;
}

extern "C" int fp64_issue_lab(int variant, int iters, float* ms) {
  double* d;
  cudaMalloc(&d, 296 * 256 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    if (variant == 0) k_lab<0><<<296, 256>>>(d, iters, 1);
    if (variant == 1) k_lab<8><<<296, 256>>>(d, iters, 1);
    if (variant == 2) k_lab<16><<<296, 256>>>(d, iters, 1);
    if (variant == 3) k_lab<32><<<296, 256>>>(d, iters, 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(ms, e0, e1);
  int e = (int)cudaGetLastError();
  cudaFree(d);
  return e;
}
