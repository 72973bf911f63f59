// K2f — fused (5-GEMM) parallel-template backward on sm_100a, dQ reduced through L2.
//
// Same VJP as K2a + K2b (parallel_bwd.cuh, the closed form of
// attention.derive_backward / graph.py:481-569), but S and dP are computed once per (key tile,
// query tile) pair: the key-tile-stationary CTA of K2a also forms dQ^T = K^T dS^T for the tile and
// adds it into an fp32 accumulator in global memory with TMA bulk reduce-adds, so the
// recompute of K2b (S = Q K^T, dP = dO V^T: 2 of K2's 7 GEMMs) disappears.  A small pass then
// scales the accumulator into bf16 dQ.  fp32 reduce-adds from different key tiles land in L2 in
// arrival order, so dQ is reproducible to fp32 rounding only (dK / dV stay bitwise deterministic);
// the split K2a/K2b pair remains the bitwise-deterministic mode (desc.bwd_mode = AF_BWD_SPLIT).
//
// One CTA per (128-key tile, b, KV head); it loops over every query head of the GQA group and
// every visible 64-row query tile — 64 rather than 128 rows so all five accumulators fit TMEM
// without aliasing (S^T x2 | dP^T | dQ^T | dV | dK = 64+64+64+64+128+128 columns) and no GEMM
// waits on the dQ drain.
//   warps 0-15  row warps: lane quarter w%4 (= key row), query columns [16*(w/4), +16);
//               P^T -> TMEM (A operand of dV), dS^T -> TMEM over its own dP^T columns (A of
//               dK) and shared memory (B operand of dQ^T)
//   warps 16-19 dQ drain: one lane quarter (32 of the 128 d rows of dQ^T) each; TMEM -> smem
//               staging -> cp.reduce.async.bulk .add.f32 (8 KB per warp and tile)
//   warp 20     TMA producer (K/V once, Q/dO/LSE/delta ring of 3)
//   warp 21     TMEM allocator + single-thread tcgen05.mma issuer
// Shared-memory bandwidth (128 B/clk) is the budget this layout is cut to: the SS GEMMs read
// 144 KB per 64-row tile, so dK takes dS^T from TMEM rather than smem (a 128-row-tile form with
// dQ^T aliased over dP^T traced at 4.7k clk per tile against 2.6k of MMA: its smem traffic,
// 512 KB per tile, set the pace).
// Per query tile the tensor pipe runs S^T = K Q^T, dP^T = V dO^T (SS, N = 64), dV += P^T dO (TS),
// dK += dS^T Q (TS), dQ^T = K^T dS^T (SS, MN-major A and B).
#pragma once
#include <cuda.h>
#include "params.h"
#include "sm100.cuh"
#include "parallel_fwd.cuh"
#include "parallel_bwd.cuh"

namespace af {

constexpr int kFusedBM = 64;  // query rows per iteration

// Developer timeline (-DAF_FUSED_TRACE): SM-clock stamps of one CTA's roles per iteration, read
// back with af_debug_fused_trace (tools/trace_fused.py).  Compiled out of the product build.
#ifdef AF_FUSED_TRACE
__device__ long long g_fused_trace[16][512];
#define FTRACE(ev, n)                                                                       \
  do {                                                                                      \
    if (blockIdx.x == 3 && blockIdx.y == 9 && (n) < 512) g_fused_trace[ev][n] = clock64();  \
  } while (0)
#else
#define FTRACE(ev, n) \
  do {                \
  } while (0)
#endif

template <int D, int DV>
struct BwdFusedSmem {
  static constexpr int kStages = 3;
  static constexpr int kKBytes = kBlockN * D * 2;
  static constexpr int kVBytes = kBlockN * DV * 2;
  static constexpr int kQBytes = kFusedBM * D * 2;
  static constexpr int kOBytes = kFusedBM * DV * 2;
  static constexpr int kDsBytes = kBlockN * kFusedBM * 2;  // dS^T [128 keys][64 queries] bf16
  static constexpr int kStgBytes = kFusedBM * D * 4;       // dQ^T staging: 4 x [64 q][32 d] fp32
  static constexpr int kKOff = 0;
  static constexpr int kVOff = kKOff + kKBytes;
  static constexpr int kQOff = kVOff + kVBytes;
  static constexpr int kOOff = kQOff + kStages * kQBytes;
  // (the epilogue stages dK / dV boxes, 4 KB per row warp, over the drained Q and dO rings)
  static constexpr int kDsOff = kOOff + kStages * kOBytes;
  static constexpr int kStgOff = kDsOff + 2 * kDsBytes;
  static constexpr int kLseOff = kStgOff + kStgBytes;
  static constexpr int kDeltaOff = kLseOff + kStages * kFusedBM * 4;
  static constexpr int kBarOff = kDeltaOff + kStages * kFusedBM * 4;
  // kv_full, full[3], empty[3], s_full[2], p_ready[2], dp_full, ds_ready[2], ds_free[2], dq_full,
  // dq_free, acc_full
  static constexpr int kNumBars = 1 + 2 * kStages + 2 + 2 + 1 + 2 + 2 + 1 + 1 + 1;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
};

// Row warps: four per TMEM lane quarter, 16 query columns each.
constexpr int kFusedRowWarps = 16;
constexpr int kFusedCols = kFusedBM / (kFusedRowWarps / 4);  // query columns per row warp
static_assert(kFusedCols == 16, "row-warp split");
constexpr int kFusedThreads = 32 * (kFusedRowWarps + 4 + 2);

// Query-row range [lo, hi) a key tile [k0, k0+128) is visible from (band mask), and whether a
// 64-row query tile x 128-key tile block is fully kept.
AF_DEVICE bool tile64_fully_kept(const MaskParams& m, int q0, int k0, int seq_q, int seq_k) {
  if (q0 + kFusedBM > seq_q || k0 + kBlockN > seq_k) return false;
  if (m.causal && k0 + kBlockN - 1 > q0 + m.diag_offset) return false;
  if (m.window > 0 && (q0 + kFusedBM - 1) + m.diag_offset - k0 >= m.window) return false;
  return true;
}

// fp32 accumulator layout: [B*Hq][q tiles of 64][D/32 chunks][64 rows][32 cols] — each drain
// warp's 8 KB partial is one contiguous bulk reduce.
__host__ __device__ inline int64_t dq_accum_offset(int64_t bh, int q_tiles64, int qt, int chunk,
                                                   int d) {
  return ((bh * q_tiles64 + qt) * (d / 32) + chunk) * (kFusedBM * 32);
}

template <int D, int DV, int kFamily, int kAct>
__global__ void __launch_bounds__(kFusedThreads, 1)
    parallel_bwd_fused_kernel(const __grid_constant__ CUtensorMap tm_q,
                              const __grid_constant__ CUtensorMap tm_k,
                              const __grid_constant__ CUtensorMap tm_v,
                              const __grid_constant__ CUtensorMap tm_do,
                              const __grid_constant__ CUtensorMap tm_dk,  // [32 rows][64] boxes
                              const __grid_constant__ CUtensorMap tm_dv,
                              const ParallelBwdParams p, const float* __restrict__ lse2,
                              const float* __restrict__ delta, int seq_q_pad,
                              float* __restrict__ dq_accum) {
  using L = BwdFusedSmem<D, DV>;
  constexpr int kStages = L::kStages;
  static_assert(D == 128 && DV % 64 == 0 && DV <= 128, "fused backward tile dims");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sO = smem + L::kOOff;
  uint8_t* sDS = smem + L::kDsOff;
  float* sLse = reinterpret_cast<float*>(smem + L::kLseOff);
  float* sDelta = reinterpret_cast<float*>(smem + L::kDeltaOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* kv_full = bars;
  uint64_t* full = kv_full + 1;
  uint64_t* empty = full + kStages;
  uint64_t* s_full = empty + kStages;   // [2]
  uint64_t* p_ready = s_full + 2;       // [2]
  uint64_t* dp_full = p_ready + 2;
  uint64_t* ds_ready = dp_full + 1;     // [2]
  uint64_t* ds_free = ds_ready + 2;     // [2]
  uint64_t* dq_full = ds_free + 2;
  uint64_t* dq_free = dq_full + 1;
  uint64_t* acc_full = dq_free + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);

  const int warp = static_cast<int>(warp_id());
  const int kt = blockIdx.x;
  const int bhk = blockIdx.y;
  const int b = bhk / p.heads_kv;
  const int hk = bhk % p.heads_kv;
  const int group = p.heads_q / p.heads_kv;
  const int k0 = kt * kBlockN;
  int qlo, qhi;
  query_band(p.mask, k0, p.seq_q, qlo, qhi);
  const int qt_lo = qlo / kFusedBM;
  const int qt_hi = (qhi > qlo) ? (qhi + kFusedBM - 1) / kFusedBM : qt_lo;
  const int tiles_per_head = qt_hi - qt_lo;
  const int niter = tiles_per_head * group;

  constexpr int kRW = kFusedRowWarps, kDrainW0 = kRW, kTmaW = kRW + 4, kMmaW = kRW + 5;
  if (warp == kTmaW && lane_id() == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&p_ready[x], kRW);
      mbar_init(&ds_ready[x], kRW);
      mbar_init(&ds_free[x], 1);
    }
    mbar_init(dp_full, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == kMmaW) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // S^T buffers [0,64) [64,128) | dP^T [128,192) | dQ^T [192,256) | dV [256,384) | dK [384,512)
  constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 192, kColDV = 256, kColDK = 384;

  if (warp == kTmaW) {
    // ───────────── TMA producer ─────────────
    if (elect_one() && niter > 0) {
      mbar_expect_tx(kv_full, L::kKBytes + L::kVBytes);
      for (int c = 0; c < D / 64; ++c)
        tma_load_4d(sK + c * (kBlockN * 128), &tm_k, kv_full, c * 64, k0, hk, b);
      for (int c = 0; c < DV / 64; ++c)
        tma_load_4d(sV + c * (kBlockN * 128), &tm_v, kv_full, c * 64, k0, hk, b);
      int hi_ = 0, qt_ = 0;
      for (int n = 0; n < niter; ++n) {
        const int s = n % kStages;
        const uint32_t ph = (n / kStages) & 1;
        const int h = hk * group + hi_;
        const int q0 = (qt_lo + qt_) * kFusedBM;
        if (++qt_ == tiles_per_head) {
          qt_ = 0;
          ++hi_;
        }
        mbar_wait(&empty[s], ph ^ 1);
        FTRACE(12, n);
        mbar_expect_tx(&full[s], L::kQBytes + L::kOBytes + 2 * kFusedBM * 4);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d_hint(sQ + s * L::kQBytes + c * (kFusedBM * 128), &tm_q, &full[s], c * 64,
                           q0, h, b, kEvictLast);
        for (int c = 0; c < DV / 64; ++c)
          tma_load_4d_hint(sO + s * L::kOBytes + c * (kFusedBM * 128), &tm_do, &full[s], c * 64,
                           q0, h, b, kEvictLast);
        const int64_t row = (static_cast<int64_t>(b) * p.heads_q + h) * seq_q_pad + q0;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(sLse + s * kFusedBM)),
            "l"(lse2 + row), "r"(kFusedBM * 4), "r"(smem_u32(&full[s]))
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(sDelta + s * kFusedBM)),
            "l"(delta + row), "r"(kFusedBM * 4), "r"(smem_u32(&full[s]))
            : "memory");
      }
    }
  } else if (warp == kMmaW) {
    // ───────────── MMA issuer ─────────────
    if (elect_one() && niter > 0) {
      constexpr uint32_t id_s = make_idesc_bf16(kBlockN, kFusedBM, false, false);  // S^T, dP^T
      constexpr uint32_t id_dv = make_idesc_bf16(kBlockN, DV, false, true);        // dV += P^T dO
      constexpr uint32_t id_dk = make_idesc_bf16(kBlockN, D, false, true);         // dK += dS^T Q
      constexpr uint32_t id_dq = make_idesc_bf16(D, kFusedBM, true, true);         // dQ^T = K^T dS^T
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ), aO = smem_u32(sO);
      const uint32_t aDS = smem_u32(sDS);
      auto kmajor = [](uint32_t base, int kk, int rows) {
        return make_sdesc(base + (kk / 4) * (rows * 128) + (kk % 4) * 32, 0, 1024);
      };
      auto wait_full = [&](int n) {
        mbar_wait(&full[n % kStages], (n / kStages) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int n) {
        const int s = n % kStages;
        const uint32_t col = kColS + (n & 1) * kFusedBM;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem + col, kmajor(aK, kk, kBlockN), kmajor(aQ + s * L::kQBytes, kk, kFusedBM),
                 id_s, kk > 0);
        mma_commit(&s_full[n & 1]);
        FTRACE(3, n);
      };
      auto issue_dp = [&](int n) {
        const int s = n % kStages;
#pragma unroll
        for (int kk = 0; kk < DV / 16; ++kk)
          mma_ss(tmem + kColDP, kmajor(aV, kk, kBlockN), kmajor(aO + s * L::kOBytes, kk, kFusedBM),
                 id_s, kk > 0);
        mma_commit(dp_full);
        FTRACE(1, n);
      };
      // Pipe order: dV(n) | dK(n) dP(n+1) dQ^T(n) | S^T(n+2).  dP(n+1) follows dK(n) (which reads
      // dS^T(n) from the dP^T columns) so the rows' dS(n+1) overlaps dQ^T(n); the S^T double
      // buffer lets S^T(n+2) follow as soon as dV(n) has read P^T(n).
      mbar_wait(kv_full, 0);
      wait_full(0);
      issue_s(0);
      issue_dp(0);
      if (niter > 1) {
        wait_full(1);
        issue_s(1);
      }
      for (int n = 0; n < niter; ++n) {
        const int s = n % kStages;
        const int buf = n & 1;
        const uint32_t ph2 = (n >> 1) & 1;
        mbar_wait(&p_ready[buf], ph2);
        FTRACE(0, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kFusedBM / 16; ++kk)
          mma_ts(tmem + kColDV, tmem + kColS + buf * kFusedBM + kFusedCols * kk,
                 make_sdesc(aO + s * L::kOBytes + kk * 16 * 128, kFusedBM * 128, 1024), id_dv,
                 (n > 0 || kk > 0));
        mbar_wait(&ds_ready[buf], ph2);
        FTRACE(2, n);
        tc_fence_after();
        const uint32_t ds = aDS + buf * L::kDsBytes;
#pragma unroll
        for (int kk = 0; kk < kFusedBM / 16; ++kk)  // A = packed dS^T over the dP^T columns
          mma_ts(tmem + kColDK, tmem + kColDP + kFusedCols * kk,
                 make_sdesc(aQ + s * L::kQBytes + kk * 16 * 128, kFusedBM * 128, 1024), id_dk,
                 (n > 0 || kk > 0));
        // stage s (Q, dO, LSE, delta of tile n) is free once dK(n) completes — its last reader
        // (traced: releasing it after dQ^T(n) left S^T(n+2) waiting on its TMA load)
        mma_commit(&empty[s]);
        // dP^T(n+1) over dS^T(n): dK(n) reads it ahead on the in-order pipe, and the rows read
        // dP^T(n) before ds_ready(n)
        if (n + 1 < niter) issue_dp(n + 1);
        if (n > 0) {
          mbar_wait(dq_free, (n - 1) & 1);  // the drain warps have read dQ^T(n-1)
          tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < kBlockN / 16; ++kk)
          mma_ss(tmem + kColDQ, make_sdesc(aK + kk * 16 * 128, kBlockN * 128, 1024),
                 make_sdesc(ds + kk * 16 * 128, kBlockN * 128, 1024), id_dq, kk > 0);
        mma_commit(dq_full);
        mma_commit(&ds_free[buf]);
        if (n + 2 < niter) {  // into buffer `buf`: P^T(n) was consumed by dV(n) above
          wait_full(n + 2);
          issue_s(n + 2);
        }
      }
      mma_commit(acc_full);
    }
  } else if (warp >= kDrainW0) {
    // ───────────── dQ drain: TMEM -> smem staging -> L2 bulk reduce-add ─────────────
    // (red.global.add.v4.f32 straight from registers measured +3.5 ms over no reduce at cfg2,
    // the TMA bulk reduce +1 ms: the per-SM reduce bursts queue behind each other in the LSU)
    const int wq = warp % 4;  // TMEM lane quarter = d rows [32 wq, 32 wq + 32)
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const int lane = static_cast<int>(lane_id());
    float* stg = reinterpret_cast<float*>(smem + L::kStgOff) + wq * (kFusedBM * 32);
    const int q_tiles64 = seq_q_pad / kFusedBM;
    int hi_ = 0, qt_ = 0;
    for (int n = 0; n < niter; ++n) {
      const int h = hk * group + hi_;
      const int qt = qt_lo + qt_;
      if (++qt_ == tiles_per_head) {
        qt_ = 0;
        ++hi_;
      }
      mbar_wait_sleep(dq_full, n & 1);
      if (lane == 0 && wq == 0) FTRACE(9, n);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      tmem_ld32(tmem + lane_base + kColDQ, r0);
      tmem_ld32(tmem + lane_base + kColDQ + 32, r1);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(dq_free);
        if (wq == 0) FTRACE(10, n);
        bulk_wait_read<0>();  // the previous reduce has finished reading the staging slice
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 32; ++q) stg[q * 32 + lane] = __uint_as_float(r0[q]);
#pragma unroll
      for (int q = 0; q < 32; ++q) stg[(32 + q) * 32 + lane] = __uint_as_float(r1[q]);
      fence_proxy_async_smem();
      __syncwarp();
#ifndef AF_FUSED_NO_REDUCE  // developer ablation: drop the L2 reduce (dQ wrong) to time the rest
      if (lane == 0) {
        float* dst = dq_accum +
                     dq_accum_offset(static_cast<int64_t>(b) * p.heads_q + h, q_tiles64, qt, wq, D);
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
            "r"(smem_u32(stg)), "r"(kFusedBM * 32 * 4)
            : "memory");
        bulk_commit();
      }
#endif
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  } else {
    // ───────────── key-row warps ─────────────
    constexpr int NC = kFusedCols;
    const int wq = warp % 4;
    const int sub = warp / 4;  // query columns [NC sub, NC sub + NC) of the 64-row tile
    const int row = wq * 32 + static_cast<int>(lane_id());
    const int j = k0 + row;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const int cb = sub * NC;
    int slope_h = -1;
    float slope = 0.0f;
    int hi_ = 0, qt_ = 0;
    for (int n = 0; n < niter; ++n) {
      const int s = n % kStages;
      const int buf = n & 1;
      const uint32_t ph2 = (n >> 1) & 1;
      const int h = hk * group + hi_;
      const int q0 = (qt_lo + qt_) * kFusedBM;
      if (++qt_ == tiles_per_head) {
        qt_ = 0;
        ++hi_;
      }
      const bool fullblk = tile64_fully_kept(p.mask, q0, k0, p.seq_q, p.seq_k);
      if constexpr (kFamily != kFamilySoftmax) {  // once per head of the group
        if (h != slope_h) {
          slope_h = h;
          slope = p.slope != nullptr ? p.slope[h] : 0.0f;
        }
      }
      const float* lse_s = sLse + s * kFusedBM + cb;
      const float* del_s = sDelta + s * kFusedBM + cb;
      mbar_wait(&full[s], (n / kStages) & 1);  // LSE / delta of this stage (already complete)
      mbar_wait(&s_full[buf], ph2);
      if (warp == 0 && lane_id() == 0) FTRACE(4, n);
      tc_fence_after();
      uint32_t pk[NC / 2], gk[NC / 2];
      uint32_t gmask;
      {
        uint32_t sr[NC];
        tmem_ld16(tmem + lane_base + kColS + buf * kFusedBM + cb, sr);
        tmem_ld_wait();
        gmask = kv_rows_p32<kFamily, kAct, NC>(p, sr, q0 + cb, j, fullblk, slope, lse_s, pk, gk);
      }
      tmem_st8(tmem + lane_base + kColS + buf * kFusedBM + cb, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&p_ready[buf]);
      if (warp == 0 && lane_id() == 0) FTRACE(5, n);

      mbar_wait(dp_full, n & 1);
      if (warp == 0 && lane_id() == 0) FTRACE(6, n);
      tc_fence_after();
      uint32_t dsk[NC / 2];
      {
        uint32_t dr[NC];
        tmem_ld16(tmem + lane_base + kColDP + cb, dr);
        tmem_ld_wait();
        make_ds<kFamily, kAct, false, NC>(pk, dr, del_s, 0.0f, gmask, dsk, gk);
      }
      // packed dS^T over this warp's own dP^T columns (A operand of dK), and the same 16 query
      // columns of this key row into the K-major SW128 tile of buffer `buf` (B operand of dQ^T)
      tmem_st8(tmem + lane_base + kColDP + cb, dsk);
      if (n >= 2) mbar_wait(&ds_free[buf], ph2 ^ 1);
      if (warp == 0 && lane_id() == 0) FTRACE(7, n);
      uint8_t* box = sDS + buf * L::kDsBytes;
#pragma unroll
      for (int q = 0; q < NC / 8; ++q) {
        const int g = cb / 8 + q;
        *reinterpret_cast<uint4*>(box + row * 128 + ((g ^ (row & 7)) << 4)) =
            make_uint4(dsk[q * 4], dsk[q * 4 + 1], dsk[q * 4 + 2], dsk[q * 4 + 3]);
      }
      fence_proxy_async_smem();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&ds_ready[buf]);
      if (warp == 0 && lane_id() == 0) FTRACE(8, n);
    }
    // ───────────── epilogue: subs 0-1 store dV rows, subs 2-3 dK rows (half the columns each)
    if (niter > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
    }
    const bool live = j < p.seq_k;
    const bool is_v = sub < 2;
    const int part = sub & 1;
    const int ncol = (is_v ? DV : D) / 2;
    const uint32_t col0 = (is_v ? kColDV : kColDK) + part * ncol;
    const float mul = is_v ? 1.0f : p.scale;
    __nv_bfloat16* dst =
        (is_v ? reinterpret_cast<__nv_bfloat16*>(p.dv) + b * p.dv_stride_b + hk * p.dv_stride_h +
                    static_cast<int64_t>(live ? j : 0) * p.dv_stride_s
              : reinterpret_cast<__nv_bfloat16*>(p.dk) + b * p.dk_stride_b + hk * p.dk_stride_h +
                    static_cast<int64_t>(live ? j : 0) * p.dk_stride_s) +
        part * ncol;
    // dK / dV through a 4 KB SW128 [32 rows][64 cols] box per warp in the drained Q / dO rings
    // and a TMA store (per-thread 16-byte row stores otherwise)
    static_assert(16 * 4096 <= kStages * (L::kQBytes + L::kOBytes), "dK / dV staging");
    const bool stage = p.dkv_tma != 0 && ncol == 64;
    uint8_t* box = sQ + warp * 4096;
    const int lr = static_cast<int>(lane_id());
#pragma unroll 1
    for (int c = 0; c < ncol / 32; ++c) {
      uint32_t r[32];
      if (niter > 0) {
        tmem_ld32(tmem + lane_base + col0 + c * 32, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) r[e] = 0u;
      }
      if (stage) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int g = c * 4 + v;
          *reinterpret_cast<uint4*>(box + lr * 128 + ((g ^ (lr & 7)) << 4)) = make_uint4(
              pack_bf16(__uint_as_float(r[v * 8 + 0]) * mul, __uint_as_float(r[v * 8 + 1]) * mul),
              pack_bf16(__uint_as_float(r[v * 8 + 2]) * mul, __uint_as_float(r[v * 8 + 3]) * mul),
              pack_bf16(__uint_as_float(r[v * 8 + 4]) * mul, __uint_as_float(r[v * 8 + 5]) * mul),
              pack_bf16(__uint_as_float(r[v * 8 + 6]) * mul, __uint_as_float(r[v * 8 + 7]) * mul));
        }
      } else if (live) {
        store_row_bf16<32>(dst + c * 32, r, mul);
      }
    }
    if (stage) {  // rows past seq_k are clipped by the map
      fence_proxy_async_smem();
      __syncwarp();
      if (lr == 0) {
        tma_store_4d(is_v ? &tm_dv : &tm_dk, box, part * ncol, k0 + wq * 32, hk, b);
        bulk_commit();
        bulk_wait<0>();
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaW) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// dQ[b, h, i, :] = scale * accumulator (bf16), eight columns per thread.
template <int D>
__global__ void __launch_bounds__(256) dq_convert_kernel(const float* __restrict__ acc,
                                                         __nv_bfloat16* __restrict__ dq,
                                                         int64_t q_sb, int64_t q_sh, int64_t q_ss,
                                                         int heads, int seq_q, int seq_q_pad,
                                                         float scale, int64_t total) {
  constexpr int kTpr = D / 8;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= total * kTpr) return;
  const int64_t rowid = t / kTpr;
  const int part = static_cast<int>(t % kTpr);
  const int64_t bh = rowid / seq_q;
  const int i = static_cast<int>(rowid % seq_q);
  const int b = static_cast<int>(bh / heads), h = static_cast<int>(bh % heads);
  const int d0 = part * 8;
  const float* src = acc + dq_accum_offset(bh, seq_q_pad / kFusedBM, i / kFusedBM, d0 / 32, D) +
                     (i % kFusedBM) * 32 + (d0 % 32);
  const float4 x = *reinterpret_cast<const float4*>(src);
  const float4 y = *reinterpret_cast<const float4*>(src + 4);
  uint4 w;
  w.x = pack_bf16(x.x * scale, x.y * scale);
  w.y = pack_bf16(x.z * scale, x.w * scale);
  w.z = pack_bf16(y.x * scale, y.y * scale);
  w.w = pack_bf16(y.z * scale, y.w * scale);
  *reinterpret_cast<uint4*>(dq + b * q_sb + h * q_sh + static_cast<int64_t>(i) * q_ss + d0) = w;
}

}  // namespace af
