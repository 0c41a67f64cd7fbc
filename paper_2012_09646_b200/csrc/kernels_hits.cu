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

// "spmv" (product, round 2): the padded non-zero split (PadPlan, spmv_common.cuh).
__global__ void __launch_bounds__(256, 4) k_spmv_pad(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                     const int* __restrict__ plan, const float* __restrict__ x,
                                                     float* __restrict__ y, long long N_) {
  (void)row_ptr;
  (void)col;  // the plan carries the (padded) graph; see above
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const PadPlan P = pad_plan(plan);
  if ((long long)P.n != N_ || P.n == 0) return;
  const int G = (int)gridDim.x * (blockDim.x >> 5);
  const int g = (int)blockIdx.x * (blockDim.x >> 5) + warp;
  const int per = (P.nc + G - 1) / G;
  const int cb = g * per, ce = min(P.nc, cb + per);
  if (cb >= ce) return;  // warp-uniform; the kernel has no CTA barriers
  const SpmvWs ws = spmv_ws(y, N_, G);
  const uint64_t pol = l2_policy_evict_first();
  auto warp_of_item = [&](int k) { return (k / kNzChunk) / per; };
  const int wsel = lane >> 3, bsh = 4 * (lane & 7);
  const unsigned lanes_below = (1u << lane) - 1u;

  const int k0w = cb * kNzChunk;
  const bool start0 = (__ldg(P.flags + (k0w >> 5)) >> (k0w & 31)) & 1u;
  int R0 = __ldg(P.rbase + cb);  // row open at the current chunk's start
  bool head_pending = !start0;   // ... which began in an earlier warp's range
  float carry = 0.f;

  NzIn cur = pad_load(P, cb, lane, pol);
  NzIn nxt = cur;
  if (cb + 1 < ce) nxt = pad_load(P, cb + 1, lane, pol);
  float v[4];
  nz_gather(cur, x, v);
  for (int c = cb; c < ce; ++c) {
    uint4 fw = cur.fw;
    if (c == cb) fw.x &= ~1u;  // the range's first item: handled by start0/head_pending
    const unsigned mine = wsel == 0 ? fw.x : (wsel == 1 ? fw.y : (wsel == 2 ? fw.z : fw.w));
    const unsigned fl = (mine >> bsh) & 0xFu;
    const int nst = __popc(fl);
    const int before = (wsel > 0 ? __popc(fw.x) : 0) + (wsel > 1 ? __popc(fw.y) : 0) +
                       (wsel > 2 ? __popc(fw.z) : 0) + __popc(mine & ((1u << bsh) - 1u));
    const int total = __popc(fw.x) + __popc(fw.y) + __popc(fw.z) + __popc(fw.w);
    const int o = R0 + before;  // row open entering the lane; ends at its first start
    float vn[4] = {0.f, 0.f, 0.f, 0.f};
    if (c + 1 < ce) {
      nz_gather(nxt, x, vn);
      cur = nxt;
      if (c + 2 < ce) nxt = pad_load(P, c + 2, lane, pol);
    }
    float run = 0.f, head = 0.f;
    bool seen = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if ((fl >> u) & 1u) {
        if (!seen) head = run;
        seen = true;
        run = 0.f;
      }
      run += v[u];
    }
    if (!seen) head = run;
    const unsigned m = __ballot_sync(0xffffffffu, nst != 0);
    float sv = nst ? run : head;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float tv = __shfl_up_sync(0xffffffffu, sv, off);
      const unsigned win = lane >= off ? (m >> (lane - off + 1)) & ((1u << off) - 1u) : 1u;
      if (win == 0u) sv += tv;
    }
    float cin = __shfl_up_sync(0xffffffffu, sv, 1);
    if (lane == 0) cin = 0.f;
    if ((m & lanes_below) == 0u) cin += carry;
    if (nst) {
      const float val = cin + head;
      if (head_pending && before == 0) {
        const int cs = warp_of_item(__ldg(P.rp2 + o));
        spmv_ws_put(ws, g, val, true);
        if (spmv_ws_arrive(ws, cs, g)) y[o] = spmv_ws_sum(ws, cs, g);
      } else {
        y[o] = val;
      }
      int j = 1;
      float r2 = 0.f;
      bool in = false;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if ((fl >> u) & 1u) {
          if (in) y[o + j++] = r2;
          in = true;
          r2 = 0.f;
        }
        r2 += v[u];
      }
    }
    const float tail_all = __shfl_sync(0xffffffffu, sv, 31);
    carry = m ? tail_all : carry + tail_all;
    if (m) head_pending = false;
    R0 += total;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = vn[u];
  }
  // the row open at the range end
  if (lane == 0) {
    const int ke = ce * kNzChunk;
    const bool ends_here = ke >= P.e2 || ((__ldg(P.flags + (ke >> 5)) >> (ke & 31)) & 1u);
    if (ends_here) {
      if (head_pending) {  // spans the whole range, ends at its end
        const int cs = warp_of_item(__ldg(P.rp2 + R0));
        spmv_ws_put(ws, g, carry, true);
        if (spmv_ws_arrive(ws, cs, g)) y[R0] = spmv_ws_sum(ws, cs, g);
      } else {
        y[R0] = carry;
      }
    } else {
      const int cs = warp_of_item(__ldg(P.rp2 + R0));
      const int cend = warp_of_item(__ldg(P.rp2 + R0 + 1) - 1);
      spmv_ws_put(ws, g, carry, false);
      if (spmv_ws_arrive(ws, cs, cend)) y[R0] = spmv_ws_sum(ws, cs, cend);
    }
  }
}

// SUM node read as the L2 norm: n = sqrt(sum v^2), fp64 accumulation.
__global__ void __launch_bounds__(256) k_l2norm(const float* __restrict__ v, RedOut* out,
                                                long long n) {
  __shared__ double sh[32];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long long done = 0;
  if (aligned16(v)) {
    const long long n4 = n >> 2;
    const float4* v4 = reinterpret_cast<const float4*>(v);
    for (long long i = tid; i < n4; i += nth) {
      float4 a = ldg_stream(v4 + i);
      acc += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
    }
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
    {"spmv", (const void*)k_spmv_pad, "const ptr, const ptr, const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_spmv_plan_kernel},
    {"l2norm", (const void*)k_l2norm, "const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_l2norm},
    {"divide", (const void*)k_divide, "const ptr, const ptr, out ptr, sint64", KF_NONE, 0, nullptr, v_divide},
};
DAGRT_REGISTER_BUILTINS(kHits);

}  // namespace dagrt
