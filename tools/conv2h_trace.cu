// Pipeline trace of the product conv2 (k_conv2_h<12,3,12>, tools only): the
// product kernel template compiled with its trace points on; SM clock of CTA
// 0 at every hand-off of its first 64 tiles (see tools/conv2h_trace.py).
#include <cstdint>
__device__ long long g_c2trace[10 * 64];
#define C2_TRACE_ON 1
#include "../paper_2012_09646_b200/csrc/kernels_conv2.cu"
namespace dagrt {  // standalone: no registry
int register_builtins(const Builtin*, int n) { return n; }
int register_builtins_ext(const Builtin*, int n, ResolveFn) { return n; }
}

extern "C" int conv2h_trace(const float* in, const float* w, float* out, int H2, int W2, long long* host_trace) {
  using namespace dagrt;
  uint64_t vals[5] = {(uint64_t)(uintptr_t)in, (uint64_t)(uintptr_t)w, (uint64_t)(uintptr_t)out, (uint64_t)H2,
                      (uint64_t)W2};
  void* tm = nullptr;
  if (int e = conv2_rows_prelaunch(vals, 5, &tm)) return e;
  using C = c2h::Cfg<12, 3, 12>;
  cudaFuncSetAttribute(k_conv2_h<12, 3, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem());
  for (int rep = 0; rep < 2; ++rep)
    k_conv2_h<12, 3, 12><<<148, C::kThreads, C::smem()>>>((const CUtensorMap*)tm, in, w, out, H2, W2);
  if (cudaError_t e = cudaDeviceSynchronize()) return (int)e;
  return (int)cudaMemcpyFromSymbol(host_trace, g_c2trace, sizeof(long long) * 640);
}
