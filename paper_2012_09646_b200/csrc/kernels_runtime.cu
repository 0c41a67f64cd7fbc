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
