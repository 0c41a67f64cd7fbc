// Experimental tensor-core conv2 shapes (libdagrt_exp.so; exp_common.cuh):
//  * conv2_ws*: the warp-specialised 3xTF32 pipeline with A_lo in TMEM and 9
//    stride-2 TMA boxes per tile (221 us per branch at its best shape);
//  * conv2_rows*: 3xTF32 with input rows staged once as pair planes, A_hi and
//    A_lo both in TMEM (not faster than conv2_ws);
//  * conv2_h*: other (rows, TMEM buffers, split warps) shapes of the product
//    kernel template.
// Design notes: kernels_conv2.cu; measurements: tools/conv2_variants.py.
#include "../conv2_tc.cuh"
#include "exp_common.cuh"

namespace dagrt {

template <int S, int NB, int SW>
__global__ void __launch_bounds__(c2ws::Cfg<S, NB, SW>::kThreads, 1)
    k_conv2_ws(const CUtensorMap* __restrict__ tmap, const float* __restrict__ in, const float* __restrict__ w,
               float* __restrict__ out, int H2, int W2) {
  using namespace c2ws;
  constexpr int kStages = S, kBufs = NB, kThreads = Cfg<S, NB, SW>::kThreads;
  constexpr uint32_t kLoBase = Cfg<S, NB, SW>::kLoBase;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* raw = sm;                               // [S][9][128 x 32 B] SW32
  unsigned char* bt = raw + kStages * kStage;            // [9][32 rows x 32 B] interleaved
  uint64_t* full = reinterpret_cast<uint64_t*>(bt + kTaps * kBTap);
  uint64_t* empty = full + kStages;
  uint64_t* loready = empty + kStages;
  uint64_t* mmadone = loready + kBufs;
  uint64_t* accempty = mmadone + kBufs;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accempty + kBufs);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  (void)in;

  // ---- setup: B = [W2_hi ; W2_lo] per tap (32 x 8 tf32), barriers, TMEM
  for (int i = t; i < 16 * 72; i += kThreads) {
    const int k = i / 72, r = i % 72, tap = r / 8, c = r % 8;
    const float x = w[i];
    uint32_t hi;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
    uint32_t lo;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(x - __uint_as_float(hi)));
    auto off = [&](int row) { return tap * kBTap + (row & 7) * 16 + (row >> 3) * 256 + (c >> 2) * 128 + (c & 3) * 4; };
    *reinterpret_cast<uint32_t*>(bt + off(k)) = hi;
    *reinterpret_cast<uint32_t*>(bt + off(16 + k)) = lo;
  }
  if (t == 0) {
    for (int q = 0; q < kStages; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, 1);
    }
    for (int b = 0; b < kBufs; ++b) {
      mbar_init(loready + b, SW);
      mbar_init(mmadone + b, 1);
      mbar_init(accempty + b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (tmap) asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;

  const int H3 = (H2 + 1) / 2, W3 = (W2 + 1) / 2;
  const int nqb = (W3 + 127) / 128;
  const long long ntiles = (long long)H3 * nqb;
  const long long G = gridDim.x;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / G + 1) : 0;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      const uint32_t tx = 9u * 32u * (uint32_t)box_rows(W2);
      for (int i = 0; i < nmine; ++i) {
        const long long tile = blockIdx.x + (long long)i * G;
        const int s = i % kStages;
        mbar_wait(empty + s, (uint32_t)(((i / kStages) & 1) ^ 1));
        C2T(0, i);
        const int p = (int)(tile / nqb), q0 = (int)(tile % nqb) * 128;
        const uint32_t bar = su32(full + s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            tma3d(su32(raw + s * kStage + (a * 3 + b) * kBox), tmap, 0, 2 * q0 + b - 1, 2 * p + a - 1, bar);
        C2T(1, i);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      for (int i = 0; i < nmine; ++i) {
        const int s = i % kStages, b = i % kBufs;
        const uint32_t pb = (uint32_t)((i / kBufs) & 1);
        mbar_wait(loready + b, pb);       // A_lo in TMEM (and the stage's TMA data seen by the split)
        C2T(2, i);
        mbar_wait(accempty + b, pb ^ 1);  // the epilogue drained this accumulator
        C2T(3, i);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d32 = tmem + b * kAccCols, d16 = d32 + 32, alo = tmem + kLoBase + b * kLoCols;
#pragma unroll
        for (int tap = 0; tap < kTaps; ++tap) {
          const uint64_t ah = desc_sw32(su32(raw + s * kStage + tap * kBox));
          const uint64_t bd = desc_plain(su32(bt + tap * kBTap));
          const uint32_t acc = tap > 0;
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(d32), "l"(ah), "l"(bd),
                       "r"(idesc(32)), "r"(acc));
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }" ::"r"(d16),
                       "r"(alo + tap * 8), "l"(bd), "r"(idesc(16)), "r"(acc));
        }
        commit(empty + s);    // stage s may be refilled
        commit(mmadone + b);  // accumulators ready; A_lo buffer free
        C2T(4, i);
      }
    }
  } else if (warp < 2 + SW) {
    // ---------------- split: lo = x - trunc_tf32(x) -> TMEM (lane = pixel row)
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const int part = (warp - 2) / 4;  // which share of the taps (SW / 4 shares)
    constexpr int kShares = SW / 4;
    constexpr int kPer = (kTaps + kShares - 1) / kShares;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int i = 0; i < nmine; ++i) {
      const int s = i % kStages, b = i % kBufs;
      mbar_wait(full + s, (uint32_t)((i / kStages) & 1));
      if (warp == 2 && lane == 0) C2T(5, i);
      mbar_wait(mmadone + b, (uint32_t)(((i / kBufs) & 1) ^ 1));  // A_lo buffer b consumed
      if (warp == 2 && lane == 0) C2T(6, i);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const unsigned char* rs = raw + s * kStage + 32 * r;
      const int sw = (r >> 2) & 1;  // 32-byte swizzle: chunk c of row r at 16 (c ^ ((r >> 2) & 1))
      const uint32_t alo = tmem + lane_off + kLoBase + b * kLoCols;
#pragma unroll
      for (int tt = 0; tt < kPer; ++tt) {
        const int tap = part * kPer + tt;
        if (tap >= kTaps) break;
        const float4 x0 = *reinterpret_cast<const float4*>(rs + tap * kBox + 16 * sw);
        const float4 x1 = *reinterpret_cast<const float4*>(rs + tap * kBox + 16 * (sw ^ 1));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(alo + tap * 8),
                     "r"(lo_bits(x0.x)), "r"(lo_bits(x0.y)), "r"(lo_bits(x0.z)), "r"(lo_bits(x0.w)),
                     "r"(lo_bits(x1.x)), "r"(lo_bits(x1.y)), "r"(lo_bits(x1.z)), "r"(lo_bits(x1.w))
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(loready + b);
      if (warp == 2 && lane == 0) C2T(7, i);
    }
  } else {
    // ---------------- epilogue: ReLU(acc_hh + acc_hl + acc_lh), 64 B per pixel
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int i = 0; i < nmine; ++i) {
      const long long tile = blockIdx.x + (long long)i * G;
      const int b = i % kBufs;
      mbar_wait(mmadone + b, (uint32_t)((i / kBufs) & 1));
      if (warp == 2 + SW && lane == 0) C2T(8, i);
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t h[16], l[16], m[16];
      const uint32_t d = tmem + lane_off + b * kAccCols;
      ld16(d, h);
      ld16(d + 16, l);
      ld16(d + 32, m);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty + b);
      const int p = (int)(tile / nqb), q = (int)(tile % nqb) * 128 + r;
      if (q < W3) {
        float4* dst = reinterpret_cast<float4*>(out + ((size_t)p * W3 + q) * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int n = 4 * k + j;
            v[j] = fmaxf(__uint_as_float(h[n]) + __uint_as_float(l[n]) + __uint_as_float(m[n]), 0.f);
          }
          dst[k] = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
      if (warp == 2 + SW && lane == 0) C2T(9, i);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

template <int R, int NB, int SW>
__global__ void __launch_bounds__(c2rows::Cfg<R, NB, SW>::kThreads, 1)
    k_conv2_rows(const CUtensorMap* __restrict__ tmap, const float* __restrict__ in, const float* __restrict__ w,
                 float* __restrict__ out, int H2, int W2) {
  using namespace c2ws;
  using c2rows::kSlot;
  using c2rows::kPlane;
  using c2rows::kPlaneStride;
  using c2rows::kABase;
  using c2rows::kACols;
  using c2rows::Tile;
  using c2rows::tile_at;
  constexpr int kThreads = c2rows::Cfg<R, NB, SW>::kThreads;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* rows = sm;                              // [R][even | odd] plane pairs, SW32
  unsigned char* bt = rows + R * kSlot;                  // [9][32 rows x 32 B] interleaved
  uint64_t* full = reinterpret_cast<uint64_t*>(bt + kTaps * kBTap);
  uint64_t* empty = full + R;
  uint64_t* loready = empty + R;
  uint64_t* mmadone = loready + NB;
  uint64_t* accempty = mmadone + NB;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accempty + NB);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  (void)in;

  for (int i = t; i < 16 * 72; i += kThreads) {
    const int k = i / 72, r = i % 72, tap = r / 8, c = r % 8;
    const float x = w[i];
    uint32_t hi, lo;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(x - __uint_as_float(hi)));
    auto off = [&](int row) { return tap * kBTap + (row & 7) * 16 + (row >> 3) * 256 + (c >> 2) * 128 + (c & 3) * 4; };
    *reinterpret_cast<uint32_t*>(bt + off(k)) = hi;
    *reinterpret_cast<uint32_t*>(bt + off(16 + k)) = lo;
  }
  if (t == 0) {
    for (int q = 0; q < R; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, SW);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(loready + b, SW);
      mbar_init(mmadone + b, 1);
      mbar_init(accempty + b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (tmap) asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;

  const int H3 = (H2 + 1) / 2, W3 = (W2 + 1) / 2;
  const int nqb = (W3 + 127) / 128;
  const long long ntiles = (long long)H3 * nqb;
  const long long per = (ntiles + gridDim.x - 1) / gridDim.x;
  const long long tb = (long long)blockIdx.x * per, te = min(ntiles, tb + per);
  const int nmine = te > tb ? (int)(te - tb) : 0;

  if (warp == 0) {
    // ---------------- TMA producer: the new input rows of each tile, in order
    if (lane == 0) {
      const uint32_t tx = 2u * kPlane;
      int rseq = 0;
      for (int i = 0; i < nmine; ++i) {
        const Tile T = tile_at(tb + i, i ? tb + i - 1 : -1, H3);
        const int q0 = T.qb * 128;
        for (int a = T.chained ? 1 : 0; a < 3; ++a, ++rseq) {
          const int slot = rseq % R;
          mbar_wait(empty + slot, (uint32_t)(((rseq / R) & 1) ^ 1));
          const uint32_t bar = su32(full + slot);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
          const int y = 2 * T.p + a - 1;
          unsigned char* dst = rows + slot * kSlot;
          // {channel 0, parity, pair, row}: even plane pairs q0.., odd plane pairs q0-1..
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
              ::"r"(su32(dst)), "l"(tmap), "r"(0), "r"(0), "r"(q0), "r"(y), "r"(bar) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
              ::"r"(su32(dst + kPlaneStride)), "l"(tmap), "r"(0), "r"(1), "r"(q0 - 1), "r"(y), "r"(bar) : "memory");
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: A_hi and A_lo from TMEM, B from shared memory
    if (lane == 0) {
      for (int i = 0; i < nmine; ++i) {
        const int b = i % NB;
        const uint32_t pb = (uint32_t)((i / NB) & 1);
        mbar_wait(loready + b, pb);
        mbar_wait(accempty + b, pb ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d32 = tmem + b * kAccCols, d16 = d32 + 32, ahi = tmem + kABase + b * kACols, alo = ahi + kLoCols;
#pragma unroll
        for (int tap = 0; tap < kTaps; ++tap) {
          const uint64_t bd = desc_plain(su32(bt + tap * kBTap));
          const uint32_t acc = tap > 0;
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }" ::"r"(d32), "r"(ahi + tap * 8),
                       "l"(bd), "r"(idesc(32)), "r"(acc));
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }" ::"r"(d16), "r"(alo + tap * 8),
                       "l"(bd), "r"(idesc(16)), "r"(acc));
        }
        commit(mmadone + b);  // accumulators ready; A buffer free
      }
    }
  } else if (warp < 2 + SW) {
    // ---------------- split: taps from the row planes -> A_hi, A_lo in TMEM
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const int part = (warp - 2) / 4;
    constexpr int kShares = SW / 4;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int rseq = 0;
    for (int i = 0; i < nmine; ++i) {
      const Tile T = tile_at(tb + i, i ? tb + i - 1 : -1, H3);
      const bool next_chained = i + 1 < nmine && tile_at(tb + i + 1, tb + i, H3).chained;
      // sequence numbers of input rows 2p-1, 2p, 2p+1
      const int s0 = T.chained ? rseq - 1 : rseq;
      const int nnew = T.chained ? 2 : 3;
      const int b = i % NB;
      mbar_wait(mmadone + b, (uint32_t)(((i / NB) & 1) ^ 1));  // A buffer b consumed by its last MMAs
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ahi = tmem + lane_off + kABase + b * kACols, alo = ahi + kLoCols;
      const int q0 = T.qb * 128;
      const bool edge = 2 * (q0 + r) + 1 >= W2;  // tap b = 2 past the row end (odd W2): zero
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int rs = s0 + a;
        const int slot = rs % R;
        mbar_wait(full + slot, (uint32_t)((rs / R) & 1));
        const unsigned char* ev = rows + slot * kSlot;
        const unsigned char* od = ev + kPlaneStride;
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          const int tap = a * 3 + bb;
          if ((tap * kShares) / kTaps != part) continue;  // this warp's share of the taps
          const int row = bb == 1 ? r : (bb == 0 ? r : r + 1);
          const unsigned char* pl = (bb == 1 ? ev : od) + 32 * row;
          const int sw = (row >> 2) & 1;
          float4 x0 = *reinterpret_cast<const float4*>(pl + 16 * sw);
          float4 x1 = *reinterpret_cast<const float4*>(pl + 16 * (sw ^ 1));
          if (bb == 2 && edge) x0 = x1 = make_float4(0.f, 0.f, 0.f, 0.f);
          auto h = [](float v) { return __float_as_uint(v) & 0xffffe000u; };
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ahi + tap * 8),
                       "r"(h(x0.x)), "r"(h(x0.y)), "r"(h(x0.z)), "r"(h(x0.w)), "r"(h(x1.x)), "r"(h(x1.y)),
                       "r"(h(x1.z)), "r"(h(x1.w))
                       : "memory");
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(alo + tap * 8),
                       "r"(lo_bits(x0.x)), "r"(lo_bits(x0.y)), "r"(lo_bits(x0.z)), "r"(lo_bits(x0.w)),
                       "r"(lo_bits(x1.x)), "r"(lo_bits(x1.y)), "r"(lo_bits(x1.z)), "r"(lo_bits(x1.w))
                       : "memory");
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(loready + b);
        // rows 2p-1 and 2p are done; 2p+1 too unless the next tile is chained
        mbar_arrive(empty + (s0 % R));
        mbar_arrive(empty + ((s0 + 1) % R));
        if (!next_chained) mbar_arrive(empty + ((s0 + 2) % R));
      }
      rseq += nnew;
    }
  } else {
    // ---------------- epilogue: ReLU(acc_hh + acc_hl + acc_lh), 64 B per pixel
    const int quarter = warp & 3, r = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int i = 0; i < nmine; ++i) {
      const Tile T = tile_at(tb + i, -1, H3);
      const int b = i % NB;
      mbar_wait(mmadone + b, (uint32_t)((i / NB) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t h[16], l[16], m[16];
      const uint32_t d = tmem + lane_off + b * kAccCols;
      ld16(d, h);
      ld16(d + 16, l);
      ld16(d + 32, m);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty + b);
      const int q = T.qb * 128 + r;
      if (q < W3) {
        float4* dst = reinterpret_cast<float4*>(out + ((size_t)T.p * W3 + q) * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int n = 4 * k + j;
            v[j] = fmaxf(__uint_as_float(h[n]) + __uint_as_float(l[n]) + __uint_as_float(m[n]), 0.f);
          }
          dst[k] = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

int conv2_tma_prelaunch(const uint64_t* vals, int nargs, void** extra);  // exp/conv2_tc_variants.cu

template <int S, int NB, int SW>
static const char* v_conv2_ws(const LaunchCheck& L) {
  using C = c2ws::Cfg<S, NB, SW>;
  return v_conv2_launch(L, C::kThreads, (unsigned)C::smem());
}

template <int R, int NB, int SW>
static const char* v_conv2_rows(const LaunchCheck& L) {
  using C = c2rows::Cfg<R, NB, SW>;
  if (const char* e = v_conv2_launch(L, C::kThreads, (unsigned)C::smem())) return e;
  // odd W2: the parity-1 pixel of the last pair lies 32 bytes past the row
  if ((L.i32(4) & 1) && !fits(L, 0, 32ull * L.i32(3) * L.i32(4) + 32)) return "odd W2 needs 32 bytes of input slack";
  return nullptr;
}

#define C2ROWS(NAME, R, NB, SW)                                                                              \
  {NAME, (const void*)k_conv2_rows<R, NB, SW>, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE,  \
   (int)c2rows::Cfg<R, NB, SW>::smem(), conv2_rows_prelaunch, v_conv2_rows<R, NB, SW>}
#define C2WS(NAME, S, NB, SW)                                                                            \
  {NAME, (const void*)k_conv2_ws<S, NB, SW>, "const ptr, const ptr, out ptr, sint32, sint32", KF_NONE, \
   (int)c2ws::Cfg<S, NB, SW>::smem(), conv2_tma_prelaunch, v_conv2_ws<S, NB, SW>}
static const Builtin kConv2Exp[] = {
    // warp-specialised TMA -> tcgen05 conv2 with A_lo in TMEM, 148 CTAs:
    // S TMA stages, NB TMEM buffers, SW split warps (threads 32 (6 + SW),
    // c2ws::Cfg<S, NB, SW>::smem() bytes of dynamic shared memory)
    C2WS("conv2_ws", 4, 2, 4),
    C2WS("conv2_ws6", 6, 2, 4),
    C2WS("conv2_ws6s8", 6, 2, 8),
    C2WS("conv2_ws6b3", 6, 3, 4),
    C2WS("conv2_ws5s8b3", 5, 3, 8),
    // row-staged: R input-row slots (8.5 KB each), NB TMEM buffers, SW split warps
    C2ROWS("conv2_rows", 12, 2, 8),
    C2ROWS("conv2_rows_s4", 12, 2, 4),
    C2ROWS("conv2_rows_r20", 20, 2, 8),
    // one fp16-split MMA per tap: R row slots, NB TMEM buffers, SW split warps
    C2H("conv2_h", 12, 3, 4),
    C2H("conv2_h_s8", 12, 3, 8),
    C2H("conv2_h_b4", 16, 4, 4),
    C2H("conv2_h_s12", 12, 3, 12),
    C2H("conv2_h_s8b2", 12, 2, 8),
    C2H("conv2_h_s8r16", 16, 3, 8),
    // more split warps / a fourth TMEM buffer (the pipeline trace of the
    // product, tools/conv2h_trace.py, puts the split stage on the critical path)
    C2H("conv2_h_s16", 12, 3, 16),
    C2H("conv2_h_s24", 12, 3, 24),
    C2H("conv2_h_s12b4", 12, 4, 12),
    C2H("conv2_h_s24b4", 12, 4, 24),
    // deeper row rings (the producer waits for row slots the split still holds)
    C2H("conv2_h_r16", 16, 3, 12),
    C2H("conv2_h_r20", 20, 3, 12),
    C2H("conv2_h_r24", 24, 3, 12),
    // A in shared memory (SS MMAs): R row slots, NB A/accumulator buffers, SW split warps
    C2HS("conv2_hs", 8, 3, 12),
    C2HS("conv2_hs_r12", 12, 3, 12),
    C2HS("conv2_hs_s8", 8, 3, 8),
    C2HS("conv2_hs_s16", 8, 3, 16),
};
DAGRT_REGISTER_EXP(kConv2Exp);

}  // namespace dagrt
