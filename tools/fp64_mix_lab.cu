// FP64-side instruction costs on sm_100a (tools only, tools/fp64_mix_lab.py):
// cycles per warp-instruction per SM sub-partition for DFMA with register
// operands, DFMA with a constant-bank operand, DMUL, DADD, MUFU.RCP64H
// (rcp.approx.ftz.f64) and I2F.F64 (+ DADD), each as 8 independent chains
// per thread at 16 warps per SM (2 CTAs x 256 threads x 148 SMs).
#include <cuda_runtime.h>
#include <stdint.h>

__constant__ double kC[4] = {0.999999, 1e-7, 0.5, 2.0};

template <int V>
__global__ void __launch_bounds__(256, 2) k_mix(double* out, int iters, double m, double c) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (V == 0) a[i] = fma(a[i], m, c);
      if (V == 1) a[i] = fma(a[i], kC[0], kC[1]);
      if (V == 2) a[i] = a[i] * m;
      if (V == 3) a[i] = a[i] + c;
      if (V == 4) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a[i]));
      if (V == 5) a[i] = a[i] + (double)(it + i);
      if (V == 6 || V == 7) a[i] = fma(a[i], m, c);
    }
    if (V == 6) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a[it & 7]));  // 8 DFMA + 1 RCP64H
    if (V == 7) {  // 8 DFMA + 1 fp32 MUFU.RCP on a value built from the double's bits
      float f = __int_as_float((__double2hiint(a[it & 7]) << 3) | 1);
      asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(f));
      a[it & 7] += (double)__float_as_int(f) * 1e-30;
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == -1.0) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

extern "C" int fp64_mix_lab(int v, int iters, float* ms) {
  double* d;
  cudaMalloc(&d, 296 * 256 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    switch (v) {
      case 0: k_mix<0><<<296, 256>>>(d, iters, 0.999999, 1e-7); break;
      case 1: k_mix<1><<<296, 256>>>(d, iters, 0.999999, 1e-7); break;
      case 2: k_mix<2><<<296, 256>>>(d, iters, 0.999999, 1e-7); break;
      case 3: k_mix<3><<<296, 256>>>(d, iters, 0.999999, 1e-7); break;
      case 4: k_mix<4><<<296, 256>>>(d, iters, 0.999999, 1e-7); break;
      case 5: k_mix<5><<<296, 256>>>(d, iters, 0.999999, 1e-7); break;
      case 6: k_mix<6><<<296, 256>>>(d, iters, 0.999999, 1e-7); break;
      case 7: k_mix<7><<<296, 256>>>(d, iters, 0.999999, 1e-7); break;
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(ms, e0, e1);
  int e = (int)cudaGetLastError();
  cudaFree(d);
  return e;
}
