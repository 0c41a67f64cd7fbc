// Shared device helpers for the sm_100a benchmark kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "builtin.h"

namespace dagrt {

constexpr int kSMs = 148;  // B200

__device__ __forceinline__ bool aligned16(const void* p) { return (((uintptr_t)p) & 15) == 0; }

// 128-bit streaming loads/stores (read-once data: do not allocate in L1).
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ldg_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ldg_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// L2 eviction-priority policies (createpolicy) and loads carrying them:
// streamed-once data evict-first, reused gather targets evict-last.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float ldg_hint(const float* p, uint64_t pol) {
  float r;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int ldg_hint(const int* p, uint64_t pol) {
  int r;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ void stg_hint(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

struct OpAdd {
  template <typename T> __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
  template <typename T> __device__ __forceinline__ T identity() const { return T(0); }
};
struct OpMax {
  template <typename T> __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
  template <typename T> __device__ __forceinline__ T identity() const { return -INFINITY; }
};
struct OpMin {
  template <typename T> __device__ __forceinline__ T operator()(T a, T b) const { return a < b ? a : b; }
  template <typename T> __device__ __forceinline__ T identity() const { return INFINITY; }
};

// Block-wide reduction in a fixed order (deterministic).  All threads get
// the result.  blockDim.x must be a multiple of 32, <= 1024.
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* sh /* >= 32 */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    T x = lane < nw ? sh[lane] : op.template identity<T>();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = op(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) sh[0] = x;
  }
  __syncthreads();
  T r = sh[0];
  __syncthreads();
  return r;
}

// Layout of a scalar-reduction output array ("out ptr" of a reduction
// vertex): the fp32 result first (what the host reads), then the grid
// arrival counter, then one fp64 partial per block.  The counter must be 0
// when the array is created; the last block resets it, so the array is
// reusable by the next launch.  Keeping the workspace inside the output
// array keeps the DAG identical to the paper's (no extra workspace edges).
struct RedOut {
  float result;
  unsigned int counter;
  double partial[1];  // [gridDim.x]
};
constexpr int kMaxRedBlocks = 1024;
constexpr size_t kRedOutBytes = 8 + 8 * (size_t)kMaxRedBlocks;

// Finish a grid-wide reduction deterministically: every block deposits its
// partial; the last block to arrive reduces partials[0..G) in index order.
// Returns true in the last block (whose threads all see *total).
template <typename Op>
__device__ __forceinline__ bool grid_finish(RedOut* out, double block_val, Op op, double identity,
                                            double* total, double* sh) {
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    out->partial[blockIdx.x] = block_val;
    __threadfence();
    unsigned prev = atomicAdd(&out->counter, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  double v = identity;
  const volatile double* part = out->partial;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v = op(v, part[i]);
  v = block_reduce(v, op, sh);
  *total = v;
  if (threadIdx.x == 0) out->counter = 0;  // reusable by the next launch
  return true;
}

}  // namespace dagrt
