// HITS kernels for sm_100a (§V-B; Fig. 6;
// reading R-HITS in DESIGN.md): 0/1 CSR SpMV, L2 norm, divide.
//
// SpMV on a power-law graph (20M rows, average degree 3, hub rows with
// ~1.5M non-zeros).  The paper used LightSpMV [31] (Kepler-era dynamic row
// distribution).  On B200 the product kernel splits the NON-ZEROS evenly
// over the warps of a persistent grid (chunks of 128, one 128-bit column
// load and 4 gathers in flight per lane), with the row structure re-encoded
// once when the graph is registered (the graph is static and resident).
// Measured bound on the HITS graph (tools/spmv_lab.py, profiles/r2_spmv_lab*):
// the 54M random 4-byte gathers alone, with the column stream, take 177 us
// (~1.1 gathers per SM per clock: one L1 wavefront per divergent lane).
// The round-1 merge-path kernel, the row-class kernel and the unpadded
// non-zero split are experimental variants (exp/spmv_variants.cu).
#include "spmv_common.cuh"

namespace dagrt {

// "spmv" (product): the padded non-zero split (PadPlan, spmv_common.cuh)
// with the segmented warp scan taken only where rows cross lanes
// (spmv_pad2_body): 255 vs 259 us per launch and 1.7% off the HITS DAG
// against the plain scan (spmv_pad_body, exp "spmv_pad"), tools/spmv_variants.py
// and tools/hits_variants.py.
__global__ void __launch_bounds__(256, 4) k_spmv_split(const int* __restrict__, const int* __restrict__,
                                                 const int* __restrict__ plan, const float* __restrict__ x,
                                                 float* __restrict__ y, long long N_) {
  spmv_pad2_body<4>(plan, x, y, N_);  // the plan carries the (padded) graph
}

// SUM node read as the L2 norm: n = sqrt(sum v^2), fp64 accumulation.
// (A cp.async.bulk-ring form, l2norm_ring.cuh / exp l2norm_t*, is faster
// only when the vector is L2-warm from repeated launches: on a vector just
// written by its producer -- the HITS DAG's case -- it measured 19.5 vs
// 18.7 us, and 25.8 vs 24.6 cold; tools/l2norm_lab.py,
// profiles/r2_l2norm_lab.json.  This register form stays.)
__global__ void __launch_bounds__(256, 8) k_l2norm(const float* __restrict__ v, RedOut* out,
                                                long long n) {
  __shared__ double sh[32];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long long done = 0;
  if (aligned16(v)) {
    const long long n4 = n >> 2;
    const float4* v4 = reinterpret_cast<const float4*>(v);
    // each float4's four squares summed in fp32 (relative 2^-23, far inside
    // the 1e-3 reduction criterion), one conversion per float4 into the fp64
    // accumulator: the per-element fp32->fp64 conversions ran on the XU pipe
    // (ncu: XU 33%) while the loop waited on memory; 32 registers keep the
    // full 8 CTAs per SM (a two-load form at 33 registers lost occupancy)
    auto sq4 = [](float4 a) { return (double)fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, a.w * a.w))); };
    long long i = tid;
    for (; i + nth < n4; i += 2 * nth) {  // two 16-byte loads in flight (latency-bound at one)
      const float4 a = ldg_stream(v4 + i), b = ldg_stream(v4 + i + nth);
      acc += sq4(a) + sq4(b);
    }
    if (i < n4) acc += sq4(ldg_stream(v4 + i));
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) acc += (double)v[i] * v[i];
  double blk = block_reduce(acc, OpAdd(), sh);
  double total;
  if (grid_finish(out, blk, OpAdd(), 0.0, &total, sh) && threadIdx.x == 0)
    out->result = (float)sqrt(total);
}

// DIV node: out = v / ||v|| (zeros if the norm is 0).
__global__ void __launch_bounds__(256) k_divide(const float* __restrict__ v,
                                                const RedOut* __restrict__ nrm,
                                                float* __restrict__ out, long long n) {
  const float s = nrm->result;
  const float is = s > 0.f ? 1.f / s : 0.f;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (aligned16(v) && aligned16(out)) {
    const long long n4 = n >> 2;
    for (long long i = tid; i < n4; i += nth) {
      float4 a = ldg_stream(reinterpret_cast<const float4*>(v) + i);
      a.x *= is; a.y *= is; a.z *= is; a.w *= is;
      reinterpret_cast<float4*>(out)[i] = a;
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) out[i] = v[i] * is;
}

// launch contracts (dagrt_launch validates them; builtin.h LaunchCheck)
static const char* v_l2norm(const LaunchCheck& L) {
  if (!fits(L, 0, 4ull * L.i(2))) return "vector needs 4 n bytes";
  return check_reduction(L, 1);
}
static const char* v_divide(const LaunchCheck& L) {
  const uint64_t n = (uint64_t)L.i(3);
  if (!fits(L, 0, 4 * n) || !fits(L, 2, 4 * n)) return "vectors need 4 n bytes";
  return fits(L, 1, 4) ? nullptr : "norm output too small";
}

static const Builtin kHits[] = {
    {"spmv", (const void*)k_spmv_split, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"l2norm", (const void*)k_l2norm, "const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_l2norm},
    {"divide", (const void*)k_divide, "const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_divide},
};
DAGRT_REGISTER_BUILTINS(kHits);

}  // namespace dagrt
