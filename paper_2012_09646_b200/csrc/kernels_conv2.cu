// DL second convolution, round 2: warp-specialised TMA -> tcgen05 pipeline
// with the A_lo operand of 3xTF32 in TENSOR MEMORY.
//
// conv2 (§V-B, Fig. 6; reading R-DL):
//   c2[p, q, n] = ReLU(sum_{a,b,c} W2[n, a, b, c] p[2p+a-1, 2q+b-1, c]),
// an implicit GEMM per 128-pixel tile: M = 128 output pixels (one output row
// segment), N = 16 channels, K = 72 = 9 taps x 8 input channels.  fp32 to
// the north_star's 1e-4 needs 3xTF32:  D = A_hi B_hi + A_hi B_lo + A_lo B_hi.
//
// Round-1 product (k_conv2_tmang, kernels_conv_tc.cu) ran 285 us per branch:
// three consumer groups of 128 threads, each with ONE TMA stage, serialised
// TMA wait -> split -> MMA -> wait -> epilogue, so ~3 tiles were in flight per
// SM and the long TMA/MMA/epilogue latencies were exposed; its A_lo tiles
// also went through shared memory twice (written by threads, read by the
// tensor core).  Here every role runs concurrently on different tiles:
//
//   warp 0      TMA producer: 9 stride-2 boxes {8 ch, 128 px, 1 row} per tile
//               (tap (a,b) = pixels 2q+b-1 of input row 2p+a-1; zero padding
//               by TMA out-of-bounds fill) into an S-stage ring (36 KB/stage);
//   warps 2-5   split: each thread (= TMEM lane = output pixel) reads its 9
//               taps from the swizzled box, forms lo = x - trunc_tf32(x) and
//               stores it into TMEM (tcgen05.st) -- A_lo never touches smem;
//   warp 1      MMA issuer (one thread): per tap an N=32 MMA A_hi x [B_hi|B_lo]
//               with A_hi = the raw box in smem (the tensor core truncates
//               fp32 to tf32, pinned by test_tensor_core_truncates_fp32_to_tf32)
//               and an N=16 MMA A_lo(TMEM) x B_hi; commits release the stage
//               and hand the accumulators to the epilogue;
//   warps 6-9   epilogue: tcgen05.ld of the 48 accumulator columns, sum of the
//               three products, ReLU, 64 B per pixel to global memory.
// NB accumulator / A_lo buffers in TMEM (512 columns) decouple MMA, split and
// epilogue; mbarriers carry every hand-off (full/empty per stage, lo-ready /
// mma-done / acc-empty per buffer).  A-from-TMEM kind::tf32 semantics are
// pinned by tools/tmem_lab.py (matches A-from-smem bit for bit).//
// The shipped kernel (registry name "conv2") is k_conv2_h<12, 3, 12>
// (conv2_tc.cuh): ONE fp16-split tcgen05 MMA per tap, input rows staged once
// as pair planes by a 4-D TMA map, 148 CTAs of 576 threads -- 169-172 us per
// branch on the full DL shapes vs 221 us for the 3xTF32 pipeline described
// above (conv2_ws) and 271 us for the round-1 product, tools/conv2_variants.py.
// Those kernels and the other shapes are experimental variants
// (exp/conv2_variants.cu, exp/conv2_tc_variants.cu in libdagrt_exp.so).
#include "conv2_tc.cuh"

namespace dagrt {


// Pre-launch hook of conv2_rows: the 4-D pair-plane tensor map of the input
// (vals = in, w, out, H2, W2), cached per (device, pointer, shape) for the
// process like the 9-box kernel's.
namespace {
struct RowsMap {
  int dev;
  uint64_t ptr;
  int h2, w2;
  void* dmap;
};
std::mutex g_rows_mu;
std::vector<RowsMap> g_rows_maps;
typedef CUresult (*EncodeFn4)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
}  // namespace

int conv2_rows_prelaunch(const uint64_t* vals, int nargs, void** extra) {
  if (nargs != 5) return (int)cudaErrorInvalidValue;
  const uint64_t ptr = vals[0];
  const int h2 = (int)(uint32_t)vals[3], w2 = (int)(uint32_t)vals[4];
  if (h2 < 1 || w2 < 1) {
    *extra = nullptr;
    return 0;
  }
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return (int)e;
  std::lock_guard<std::mutex> lk(g_rows_mu);
  for (const RowsMap& e : g_rows_maps)
    if (e.dev == dev && e.ptr == ptr && e.h2 == h2 && e.w2 == w2) {
      *extra = e.dmap;
      return 0;
    }
  static EncodeFn4 encode = nullptr;
  if (!encode) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fp)
      return (int)cudaErrorNotSupported;
    encode = (EncodeFn4)fp;
  }
  if (ptr & 15) return (int)cudaErrorMisalignedAddress;
  CUtensorMap m;
  const cuuint64_t pairs = (cuuint64_t)((w2 + 1) / 2);
  const cuuint64_t dims[4] = {8, 2, pairs, (cuuint64_t)h2};
  const cuuint64_t strides[3] = {32, 64, (cuuint64_t)w2 * 32};  // bytes, dims 1..3
  const cuuint32_t box[4] = {8, 1, 129, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)(uintptr_t)ptr, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return (int)cudaErrorInvalidValue;
  void* d = nullptr;
  if (cudaError_t e = cudaMalloc(&d, sizeof(CUtensorMap))) return (int)e;
  if (cudaError_t e = cudaMemcpy(d, &m, sizeof(CUtensorMap), cudaMemcpyHostToDevice)) return (int)e;
  g_rows_maps.push_back(RowsMap{dev, ptr, h2, w2, d});
  *extra = d;
  return 0;
}

static const Builtin kConv2[] = {
    // PRODUCT (round 2): one fp16-split MMA per tap, rows staged once, 12 split
    // warps (148 CTAs of 576 threads, c2h::Cfg<12, 3, 12>::smem() bytes)
    C2H("conv2", 12, 3, 12),
};
DAGRT_REGISTER_BUILTINS(kConv2);

}  // namespace dagrt
