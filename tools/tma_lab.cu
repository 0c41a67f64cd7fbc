// TMA laboratory (tools only): how fast can one CTA per SM stream the conv2
// input through TMA boxes, with no compute?  MODE 0: the product's 9 boxes per
// tile {8 ch, 128 px with TRAVERSAL STRIDE 2, 1 row}; MODE 1: the same bytes
// as 9 contiguous boxes {8, 128, 1} (no element stride); MODE 2: 6 contiguous
// boxes {8, 129, 1} per tile (3 input rows x 2 halves, the row-staging
// alternative).  A producer thread keeps S stages in flight; a consumer warp
// only waits for each stage and releases it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const void* m, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}

template <int MODE, int S>
__global__ void __launch_bounds__(64, 1) k_tma(const CUtensorMap* tmap, int H2, int W2) {
  extern __shared__ unsigned char raw_[];
  unsigned char* raw = (unsigned char*)(((uintptr_t)raw_ + 1023) & ~(uintptr_t)1023);
  constexpr int kStage = 9 * 4096;
  __shared__ uint64_t full[S], empty[S];
  const int t = threadIdx.x;
  if (t == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(empty + i)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int H3 = (H2 + 1) / 2, W3 = (W2 + 1) / 2, nqb = (W3 + 127) / 128;
  const long long ntiles = (long long)H3 * nqb;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  if (t == 0) {
    for (int i = 0; i < nmine; ++i) {
      const long long tile = blockIdx.x + (long long)i * gridDim.x;
      const int s = i % S;
      mwait(empty + s, ((i / S) & 1) ^ 1);
      const int p = (int)(tile / nqb), q0 = (int)(tile % nqb) * 128;
      const uint32_t bar = su32(full + s);
      const uint32_t tx = MODE == 2 ? 6u * 129u * 32u : 9u * 4096u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
      if (MODE == 2) {
        for (int a = 0; a < 3; ++a)
          for (int h = 0; h < 2; ++h)
            tma3(su32(raw + s * kStage + (a * 2 + h) * 129 * 32), tmap, 0, 2 * q0 - 1 + 129 * h, 2 * p + a - 1, bar);
      } else {
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b)
            tma3(su32(raw + s * kStage + (a * 3 + b) * 4096), tmap, 0, MODE == 0 ? 2 * q0 + b - 1 : q0 + 128 * b,
                 2 * p + a - 1, bar);
      }
    }
  } else if (t == 32) {
    for (int i = 0; i < nmine; ++i) {
      const int s = i % S;
      mwait(full + s, (i / S) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)) : "memory");
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
}  // namespace

extern "C" float tma_lab(int mode, int stages, const float* in, int H2, int W2, int reps) {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  CUtensorMap m;
  const cuuint64_t dims[3] = {8, (cuuint64_t)W2, (cuuint64_t)H2};
  const cuuint64_t strides[2] = {32, (cuuint64_t)W2 * 32};
  const cuuint32_t box[3] = {8, mode == 0 ? 256u : (mode == 1 ? 128u : 129u), 1};
  const cuuint32_t estr[3] = {1, mode == 0 ? 2u : 1u, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)in, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          mode == 2 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -2.f;
  void* dm = nullptr;
  cudaMalloc(&dm, sizeof(m));
  cudaMemcpy(dm, &m, sizeof(m), cudaMemcpyHostToDevice);
  const size_t smem = 1024 + (size_t)stages * 9 * 4096;
  auto launch = [&]() {
#define L(MO, S_)                                                                                    \
  if (mode == MO && stages == S_) {                                                                  \
    cudaFuncSetAttribute(k_tma<MO, S_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    k_tma<MO, S_><<<148, 64, smem>>>((const CUtensorMap*)dm, H2, W2);                                \
  }
    L(0, 4) L(0, 6) L(1, 4) L(1, 6) L(2, 4) L(2, 6)
#undef L
  };
  launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(dm);
  if (cudaGetLastError() != cudaSuccess) return -1.f;
  return ms / reps;
}
