// Host cost per call of the CUDA primitives the scheduler issues per vertex,
// against dagrt_launch itself (through the C ABI, no Python).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -Iinclude tools/launch_cost.cu \
//        -Lpaper_2012_09646_b200 -ldagrt -lcuda -o /tmp/launch_cost && \
//   LD_LIBRARY_PATH=paper_2012_09646_b200 /tmp/launch_cost
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "dagrt.h"

__global__ void k_read(const float* src, volatile float* dst, int n) {
  if (threadIdx.x < n) dst[threadIdx.x] = src[threadIdx.x];
}

__global__ void k_nop(const float* a, float* b, long long n) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && n < 0) b[0] = a[0];
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const int N = 4000;
  float *a, *b;
  cudaMalloc(&a, 4096);
  cudaMalloc(&b, 4096);
  cudaMemset(a, 0, 4096);
  cudaStream_t s, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  long long n = 1024;
  void* args[] = {&a, &b, &n};
  std::vector<cudaEvent_t> ev(N);
  for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  CUfunction f;
  cudaGetFuncBySymbol(&f, (const void*)k_nop);
  auto bench = [&](const char* name, auto fn) {
    for (int i = 0; i < 200; ++i) fn(i);
    cudaDeviceSynchronize();
    double t0 = now_us();
    for (int i = 0; i < N; ++i) fn(i);
    double t1 = now_us();
    cudaDeviceSynchronize();
    printf("{\"op\": \"%s\", \"us_per_call\": %.3f}\n", name, (t1 - t0) / N);
  };
  bench("cudaLaunchKernel", [&](int) { cudaLaunchKernel((const void*)k_nop, 1, 32, args, 0, s); });
  bench("cuLaunchKernel", [&](int) { cuLaunchKernel(f, 1, 1, 1, 32, 1, 1, 0, (CUstream)s, args, nullptr); });
  bench("cudaEventRecord", [&](int i) { cudaEventRecord(ev[i % N], s); });
  bench("cuEventRecord", [&](int i) { cuEventRecord((CUevent)ev[i % N], (CUstream)s); });
  bench("cudaStreamWaitEvent", [&](int i) { cudaStreamWaitEvent(s2, ev[i % N], 0); });
  bench("launch+record", [&](int i) {
    cudaLaunchKernel((const void*)k_nop, 1, 32, args, 0, s);
    cudaEventRecord(ev[i % N], s);
  });
  bench("cu launch+record", [&](int i) {
    cuLaunchKernel(f, 1, 1, 1, 32, 1, 1, 0, (CUstream)s, args, nullptr);
    cuEventRecord((CUevent)ev[i % N], (CUstream)s);
  });

  // dagrt: a dependent chain a -> b -> a (one stream), then fan-out (new streams)
  dagrt_config cfg = {DAGRT_PARALLEL_ASYNC, 1, 0, 0, DAGRT_BACKEND_CUDA, 0};
  dagrt_ctx c;
  if (dagrt_create(0, &cfg, &c)) { printf("create failed\n"); return 1; }
  dagrt_array A, B;
  dagrt_array_register(c, a, nullptr, 4096, &A);
  dagrt_array_register(c, b, nullptr, 4096, &B);
  dagrt_kernel k;
  // a built-in kernel (this executable's own kernels belong to another cudart instance)
  if (dagrt_kernel_lookup(c, "square", &k)) { printf("lookup failed\n"); return 1; }
  dagrt_arg ab[3], ba[3];
  ab[0].array = A; ab[1].array = B; ab[2].i64 = n;
  ba[0].array = B; ba[1].array = A; ba[2].i64 = n;
  dagrt_dim3 g1 = {1, 1, 1}, b1 = {32, 1, 1};
  bench("dagrt_launch chain", [&](int i) {
    if (dagrt_launch(c, k, g1, b1, 0, (i & 1) ? ba : ab, 3)) { printf("%s\n", dagrt_last_error(c)); exit(1); }
  });
  dagrt_sync(c);
  float z;
  bench("dagrt chain+host_read/8", [&](int i) {
    dagrt_launch(c, k, g1, b1, 0, (i & 1) ? ba : ab, 3);
    if ((i & 7) == 7) dagrt_host_read(c, A, 0, 4, &z);
  });
  dagrt_sync(c);
  bench("cudaMemcpyAsync D2H 4B + sync", [&](int) {
    static float* hp = nullptr;
    if (!hp) cudaMallocHost(&hp, 64);
    cudaMemcpyAsync(hp, a, 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  });
  bench("launch + D2H 4B + sync", [&](int) {
    static float* hp = nullptr;
    if (!hp) cudaMallocHost(&hp, 64);
    cudaLaunchKernel((const void*)k_nop, 1, 32, args, 0, s);
    cudaMemcpyAsync(hp, a, 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  });
  bench("launch + sync", [&](int) {
    cudaLaunchKernel((const void*)k_nop, 1, 32, args, 0, s);
    cudaStreamSynchronize(s);
  });
  float *hm = nullptr, *dm = nullptr;
  cudaHostAlloc(&hm, 64, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&dm, hm, 0);
  bench("launch + read kernel to mapped + sync", [&](int) {
    cudaLaunchKernel((const void*)k_nop, 1, 32, args, 0, s);
    k_read<<<1, 32, 0, s>>>(a, dm, 1);
    cudaStreamSynchronize(s);
  });
  bench("launch + read kernel to mapped + spin", [&](int i) {
    cudaLaunchKernel((const void*)k_nop, 1, 32, args, 0, s);
    hm[1] = -1.f;
    k_read<<<1, 32, 0, s>>>(a, dm, 2);
    while (((volatile float*)hm)[1] == -1.f) {}
  });
  // VEC (Fig. 4) through the C ABI, no Python: 2 squares + reduce_diff + host
  // read of z, N = 1M, resident inputs -- the C-level floor of bench.py's VEC
  {
    const long long N = 1000000;
    float *x, *y, *x1, *y1;
    void* z;
    cudaMalloc(&x, N * 4); cudaMalloc(&y, N * 4); cudaMalloc(&x1, N * 4); cudaMalloc(&y1, N * 4);
    cudaMalloc(&z, 8 + 8 * 1024);
    cudaMemset(x, 0, N * 4); cudaMemset(y, 0, N * 4); cudaMemset(z, 0, 8 + 8 * 1024);
    cudaDeviceSynchronize();
    dagrt_array X, Y, X1, Y1, Z;
    dagrt_array_register(c, x, nullptr, N * 4, &X);
    dagrt_array_register(c, y, nullptr, N * 4, &Y);
    dagrt_array_register(c, x1, nullptr, N * 4, &X1);
    dagrt_array_register(c, y1, nullptr, N * 4, &Y1);
    dagrt_array_register(c, z, nullptr, 8 + 8 * 1024, &Z);
    dagrt_kernel ksq, kred;
    dagrt_kernel_lookup(c, "square", &ksq);
    dagrt_kernel_lookup(c, "reduce_diff", &kred);
    const unsigned g = (unsigned)((N + 2047) / 2048);  // programs/vec_bs.py grid_1d(n, 256, 8)
    dagrt_arg ax[3], ay[3], ar[4];
    ax[0].array = X; ax[1].array = X1; ax[2].i64 = N;
    ay[0].array = Y; ay[1].array = Y1; ay[2].i64 = N;
    ar[0].array = X1; ar[1].array = Y1; ar[2].array = Z; ar[3].i64 = N;
    dagrt_dim3 G = {g, 1, 1}, Gr = {g < 1024 ? g : 1024, 1, 1}, B = {256, 1, 1};
    float zz;
    bench("VEC DAG via C ABI (3 launches + host read)", [&](int) {
      dagrt_launch(c, ksq, G, B, 0, ax, 3);
      dagrt_launch(c, ksq, G, B, 0, ay, 3);
      dagrt_launch(c, kred, Gr, B, 0, ar, 4);
      dagrt_host_read(c, Z, 0, 4, &zz);
    });
    if (const char* e = dagrt_last_error(c)) if (*e) printf("dagrt: %s\n", e);
  }
  dagrt_destroy(c);
  return 0;
}
