// K3b — MLA backward on sm_100a (DeepSeek-V2 latent attention: Dqk = 576, Dv = 512, one KV head
// shared by every query head, V = K[:, :512]).
//
// The VJP is the softmax-family closed form of K2 with the latent aliasing of
// SURVEY §8c(1):  dKV = sum_h (tau dS_h^T Q_h) + [sum_h P_h^T dO_h, 0].
//
// Why not K2's fused key-/query-stationary kernels: a 128 x 576 fp32 accumulator (288 KB) does not
// fit in TMEM (256 KB), and a 128-row Q/dO tile pair is 272 KB of shared memory.  Instead the
// backward is split into dense tensor-core phases that each fit the SM:
//   1. scores   (key-tile stationary, the key tile in TMEM as the MMA's A operand, Q/dO streamed
//               in 64-column boxes through a 12-stage ring): S^T = K Q^T, dP^T = V dO^T; one
//               thread per key row writes P^T = exp(S tau - LSE) and dS'^T = tau P (dP - D) as
//               bf16 rows [B*H, k_pad, q_pad] to HBM (only the causal blocks; padded rows/cols
//               written as zeros).
//   2. dQ GEMM  (query-tile stationary): dQ[:, n0:n0+N] = dS' K[:, n0:n0+N], N = 512 then 64.
//   3. dKV GEMM (key-tile stationary, one CTA per head group): dKV[:, n0:n0+N] =
//               sum_{h in group, q tiles} dS'^T Q[:, n0:] + P^T dO[:, n0:] (dO only below 512);
//               fp32 partials per head group, summed in group order by a reduce kernel.
// No atomics: results are bitwise deterministic.
//
// The same phases serve every head-dim pair K2 cannot hold in TMEM (K2a needs S^T | dP^T | dV | dK
// = 256 + Dv + Dqk columns): softmax-deepseek (192, 128) and softmax-diff (128, 256) run them with
// separate K and V tiles, GQA head groups, and dK / dV accumulated by their own GEMMs.
#pragma once
#include <cuda.h>
#include "params.h"
#include "sm100.cuh"
#include "parallel_fwd.cuh"

namespace af {

constexpr int kMbDqk = 576;
constexpr int kMbDv = 512;

struct MlaBwdParams {
  int batch, heads, heads_kv, seq_q, seq_k, q_pad, k_pad;
  float scale, scale_log2;
  MaskParams mask;
  const float* lse2;   // [B*H, q_pad] LSE * log2(e) (+inf for padded / fully-masked rows)
  const float* delta;  // [B*H, q_pad] rowsum(dO * O)
  __nv_bfloat16* p;    // [B*H, q_pad, k_pad]
  __nv_bfloat16* ds;   // [B*H, q_pad, k_pad]  (tau folded in)
  // dQ output (bf16, q strides) and dKV partials fp32 [G, B, k_pad, 576]
  void* dq;
  int64_t dq_sb, dq_sh, dq_ss;
  float* dkv_part;   // fp32 partials [G, B*Hkv, k_pad, width] of the key-side GEMM
  int groups;        // head chunks per KV head (partials summed in chunk order)
  int part_width;    // columns of one partial row (576 for MLA, Dqk for dK, Dv for dV)
  int dq_tma;        // pair dQ GEMM: dQ leaves through its store map (TMA stores)
  int part_tma;      // pair key-side GEMMs: fp32 partials leave through their store map
};

// ═══════════════════════════════ 1. scores ═══════════════════════════════
// Developer wait accounting (-DAF_SCORES_TRACE): per CTA (the first 256), SM cycles the MMA thread
// spends in its waits and in total, and the same for key-row warp 0; read with
// af_debug_scores_trace (tools/trace_scores.py).
#ifdef AF_SCORES_TRACE
__device__ long long g_scores_trace[256][8];
#define SC_T0() long long sc_t = clock64()
#define SC_ACC(slot, expr)                                                   \
  do {                                                                       \
    const long long sc_a = clock64();                                        \
    expr;                                                                    \
    if (blockIdx.x < 256) g_scores_trace[blockIdx.x][slot] += clock64() - sc_a; \
  } while (0)
#define SC_TOTAL(slot) \
  if (blockIdx.x < 256) g_scores_trace[blockIdx.x][slot] = clock64() - sc_t
#else
#define SC_T0() \
  do {          \
  } while (0)
#define SC_ACC(slot, expr) expr
#define SC_TOTAL(slot) \
  do {                 \
  } while (0)
#endif

template <int D, int DV, bool kShared>
struct MlaScoresSmem {
  static constexpr int kBox = 128 * 128;              // [128 rows][64 bf16] key-tile box
  static constexpr int kSlot = 64 * 128;              // [64 rows][64 bf16] half Q / dO box
  static constexpr int kKB = D / 64, kVB = DV / 64;   // boxes per K / V row tile
  // The key tile's operand boxes live in TMEM (A of tcgen05.mma from TMEM: 32 columns per 64-wide
  // box, eight slots over columns [256, 512)) — K boxes first, then (separate V) the V boxes.
  // K boxes beyond the eight slots (MLA: the 64 rope columns) stay resident in shared memory.
  static constexpr int kKT = kShared ? (kKB < 8 ? kKB : 8) : kKB;  // K boxes in TMEM
  static constexpr int kKS = kKB - kKT;                             // K boxes in smem
  static constexpr int kStg = kKT + (kShared ? 0 : kVB);            // boxes staged into TMEM
  static_assert(kStg <= 8 && (!kShared || kVB <= kKT), "operand boxes must fit the TMEM slots");
  // ring of half boxes (this CTA's 64 of a Q / dO box's 128 query rows): all the shared memory
  // the resident boxes leave — the ring depth sets the bytes in flight
  // + one 4 KB staging box per key-row warp for the TMA stores of its P^T / dS'^T rows
  static constexpr int kOutBytes = 8 * 4096;
  static constexpr int kStagesFit = (225 * 1024 - kKS * kBox - kOutBytes - 4608) / kSlot;
  static constexpr int kStages = kStagesFit > 24 ? 24 : kStagesFit;
  static_assert(kStages >= 2 * kStg + 2, "the staged operand boxes occupy the top ring slots");
  static constexpr int kStgBase = kStages - 2 * kStg;  // first ring slot holding a staged box
  static constexpr int kKsOff = 0;
  static constexpr int kOutOff = kKsOff + kKS * kBox;
  static constexpr int kRingOff = kOutOff + kOutBytes;
  // row statistics (LSE*log2e, D) of a query tile: a ring of 4 — the producer loads tile n+2's
  // while the rows may still be on tile n (with 2 slots it stalled the Q / dO stream behind them)
  static constexpr int kStatSlots = 4;
  static constexpr int kStatOff = kRingOff + kStages * kSlot;  // [kStatSlots][2][128] fp32
  static constexpr int kBarOff = kStatOff + kStatSlots * 2 * 128 * 4;
  // k_full, k_ready, full[S], empty[S], stat_full[4], stat_empty[4], s_full, s_free, dp_full,
  // dp_free
  static constexpr int kNumBars = 2 + 2 * kStages + 2 * kStatSlots + 4;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
};

__host__ __device__ inline int mla_q_tile_lo(const MaskParams& m, int k0) {
  // first 128-row query tile that sees key k0 under a top-left causal band
  return m.causal ? max(0, k0 - m.diag_offset) / 128 : 0;
}

// Key-tile stationary, transposed, on a CTA pair: S^T = K Q^T and dP^T = V dO^T as M = 256
// tcgen05.mma over two key tiles (the pair's leader issues; each CTA's key tile is its A operand,
// read from its own TMEM), N = 128 query rows of which each CTA streams 64 — so every Q / dO byte
// is fetched from L2 once per two key tiles, and a 24-slot ring of half boxes is in flight per SM
// (the single-CTA form streamed whole boxes per key tile: L2-throughput and latency bound, ncu
// tensor pipe 31 -> 40 % active).
// TMEM (each CTA): S^T [0, 128) | dP^T [128, 256) | operand boxes [256, 512).  One thread per key
// row writes P^T and dS'^T rows: [B*H, k_pad, q_pad] bf16 (the GEMMs read them in this layout).
// Both CTAs walk the leader's query tiles; the second key tile's extra (diagonal-below) tile is
// fully masked and written as zeros — the paired GEMMs read that block.
template <int D, int DV, bool kShared>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    mla_bwd_scores_kernel(const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v,
                          const __grid_constant__ CUtensorMap tm_pst,   // P^T store, [32][64] boxes
                          const __grid_constant__ CUtensorMap tm_dsst,  // dS'^T store
                          const MlaBwdParams p) {
  using L = MlaScoresSmem<D, DV, kShared>;
  constexpr int kStages = L::kStages;
  constexpr int kKB = L::kKB, kVB = L::kVB, kPerTile = kKB + kVB;
  constexpr int kKT = L::kKT, kStg = L::kStg, kStgBase = L::kStgBase;
  constexpr int kSS = L::kStatSlots;
  constexpr uint32_t kColS = 0, kColDP = 128, kColOp = 256;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sKs = smem + L::kKsOff;
  uint8_t* sRing = smem + L::kRingOff;
  float* sStat = reinterpret_cast<float*>(smem + L::kStatOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* k_full = bars;
  uint64_t* k_ready = bars + 1;
  uint64_t* full = bars + 2;
  uint64_t* empty = full + kStages;
  uint64_t* stat_full = empty + kStages;
  uint64_t* stat_empty = stat_full + kSS;
  uint64_t* s_full = stat_empty + kSS;
  uint64_t* s_free = s_full + 1;
  uint64_t* dp_full = s_free + 1;
  uint64_t* dp_free = dp_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);

  const int warp = static_cast<int>(warp_id());
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  // CTA order (b, h)-major with the key tiles of one head adjacent (pairs = even / odd key tile),
  // and every CTA walks its query tiles from the last one down: the CTAs of one head stream the
  // same Q / dO tiles at the same time (one HBM read, L2 for the other key tiles).
  const int k_tiles = p.k_pad / 128;  // even (k_pad is padded to 256)
  const int kt = static_cast<int>(blockIdx.x) % k_tiles;
  const int bh = static_cast<int>(blockIdx.x) / k_tiles;
  const int b = bh / p.heads, h = bh % p.heads;
  const int hk = h / (p.heads / p.heads_kv);
  const int k0 = kt * 128;
  const int q_tiles = p.q_pad / 128;
  const int nq = q_tiles - mla_q_tile_lo(p.mask, (kt & ~1) * 128);  // the leader's tiles

  if (warp == 8 && lane_id() == 0) {
    mbar_init(k_full, 1);
    mbar_init(k_ready, leader ? 16 : 8);  // the leader's MMA needs both CTAs' operand boxes
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int t = 0; t < kSS; ++t) {
      mbar_init(&stat_full[t], 1);
      mbar_init(&stat_empty[t], 8);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 16);  // (leader's: both CTAs' row warps)
    mbar_init(dp_full, 1);
    mbar_init(dp_free, 16);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any cross-CTA arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t k_ready_l = peer_addr(k_ready, 0), s_free_l = peer_addr(s_free, 0),
                 dp_free_l = peer_addr(dp_free, 0);

  if (warp == 8) {
    // ───────────── TMA producer (each CTA: its key tile, its half of every Q / dO box) ─────────────
    if (elect_one() && nq > 0) {
      mbar_expect_tx(k_full, (L::kKS + kStg) * L::kBox);
      for (int c = kKT; c < kKB; ++c)
        tma_load_4d(sKs + (c - kKT) * L::kBox, &tm_k, k_full, c * 64, k0, hk, b);
      for (int x = 0; x < kStg; ++x) {
        uint8_t* dst = sRing + (kStgBase + 2 * x) * L::kSlot;
        if (x < kKT)
          tma_load_4d(dst, &tm_k, k_full, x * 64, k0, hk, b);
        else
          tma_load_4d(dst, &tm_v, k_full, (x - kKT) * 64, k0, hk, b);
      }
      bool staged = true;  // the top slots still hold the staged boxes
      int slot = 0;
      uint32_t ph = 0;
      for (int n = 0; n < nq; ++n) {
        const int q0 = (q_tiles - 1 - n) * 128;
        const int t = n % kSS;
        mbar_wait(&stat_empty[t], ((n / kSS) & 1) ^ 1);
        mbar_expect_tx(&stat_full[t], 2 * 128 * 4);
        const int64_t row = static_cast<int64_t>(bh) * p.q_pad + q0;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(sStat + t * 256)),
            "l"(p.lse2 + row), "r"(128 * 4), "r"(smem_u32(&stat_full[t]))
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(sStat + t * 256 + 128)),
            "l"(p.delta + row), "r"(128 * 4), "r"(smem_u32(&stat_full[t]))
            : "memory");
        const int r0 = q0 + static_cast<int>(rank) * 64;  // this CTA's 64 query rows
        for (int c = 0; c < kPerTile; ++c) {
          if (staged && slot >= kStgBase) {
            mbar_wait(k_ready, 0);  // the row warps have copied the staged boxes into TMEM
            staged = false;
          }
          mbar_wait(&empty[slot], ph ^ 1);  // the pair's MMA has read this slot in both CTAs
          if (leader) mbar_expect_tx(&full[slot], 2 * L::kSlot);
          const uint32_t fl = peer_addr(&full[slot], 0);
          if (c < kKB)
            tma_load_4d_pair(sRing + slot * L::kSlot, &tm_q, fl, c * 64, r0, h, b);
          else
            tma_load_4d_pair(sRing + slot * L::kSlot, &tm_do, fl, (c - kKB) * 64, r0, h, b);
          if (++slot == kStages) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 9) {
    // ───────────── MMA issuer (the leader, for both CTAs) ─────────────
    if (leader && nq > 0 && elect_one()) {
      constexpr uint32_t id = make_idesc_bf16(256, 128, false, false);
      const uint32_t aR = smem_u32(sRing), aKs = smem_u32(sKs);
      SC_T0();
      mbar_wait(k_full, 0);   // the smem-resident K boxes (the peer's: behind its k_ready)
      SC_ACC(0, mbar_wait(k_ready, 0));  // both CTAs' TMEM operand boxes
      tc_fence_after();
      int slot = 0;
      uint32_t ph = 0;
      for (int n = 0; n < nq; ++n) {
        // S^T = K Q^T once both CTAs' row warps have read S^T(n-1)
        if (n > 0) {
          SC_ACC(1, mbar_wait(s_free, (n - 1) & 1));
          tc_fence_after();
        }
        // (box loops fully unrolled: with the TS / SS choice a runtime branch, the compiler
        // wrapped every MMA in an ELECT waterfall and the single issuing thread fell behind)
#pragma unroll
        for (int c = 0; c < kKB; ++c) {
          SC_ACC(2, mbar_wait(&full[slot], ph));
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t bd = make_sdesc(aR + slot * L::kSlot + kk * 32, 0, 1024);
            const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
            if (c < kKT)
              mma_ts_pair(tmem + kColS, tmem + kColOp + c * 32 + kk * 8, bd, id, acc);
            else
              mma_ss_pair(tmem + kColS, make_sdesc(aKs + (c - kKT) * L::kBox + kk * 32, 0, 1024),
                          bd, id, acc);
          }
          mma_commit_pair(&empty[slot]);
          if (++slot == kStages) {
            slot = 0;
            ph ^= 1;
          }
        }
        mma_commit_pair(s_full);
        // dP^T = V dO^T once both CTAs have read dP^T(n-1)  (MLA: V = K boxes 0 .. Dv/64-1)
        if (n > 0) {
          SC_ACC(3, mbar_wait(dp_free, (n - 1) & 1));
          tc_fence_after();
        }
#pragma unroll
        for (int c = 0; c < kVB; ++c) {
          SC_ACC(2, mbar_wait(&full[slot], ph));
          tc_fence_after();
          const uint32_t a = tmem + kColOp + (kShared ? c : kKT + c) * 32;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts_pair(tmem + kColDP, a + kk * 8,
                        make_sdesc(aR + slot * L::kSlot + kk * 32, 0, 1024), id,
                        (c > 0 || kk > 0) ? 1u : 0u);
          mma_commit_pair(&empty[slot]);
          if (++slot == kStages) {
            slot = 0;
            ph ^= 1;
          }
        }
        mma_commit_pair(dp_full);
      }
      SC_TOTAL(4);
    }
  } else if (nq > 0) {
    // ───────────── key-row warps: P^T and dS'^T rows ─────────────
    const int wq = warp % 4, half = warp / 4;  // TMEM lane quarter, 64-query column half
    const int jr = wq * 32 + static_cast<int>(lane_id());
    const int j = k0 + jr;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    // stage the key tile's operand boxes into TMEM: row jr of box x -> columns [32 x, +32)
    mbar_wait(k_full, 0);
    for (int x = half; x < kStg; x += 2) {
      const uint8_t* box = sRing + (kStgBase + 2 * x) * L::kSlot;
      uint32_t v[32];
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const uint4 q = *reinterpret_cast<const uint4*>(box + jr * 128 + ((g ^ (jr & 7)) << 4));
        v[g * 4 + 0] = q.x;
        v[g * 4 + 1] = q.y;
        v[g * 4 + 2] = q.z;
        v[g * 4 + 3] = q.w;
      }
      tmem_st32(tmem + lane_base + kColOp + x * 32, v);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane_id() == 0) {
      if (!leader) mbar_arrive(k_ready);  // this CTA's producer may reuse the staging slots
      mbar_arrive_cluster(k_ready_l);     // the leader's MMA may read this CTA's boxes
    }

    const float sc = p.scale;
    // this warp's 32 key rows x 64 query columns go out through a swizzled 4 KB box and a TMA
    // store (per-thread 16-byte stores to 32 different rows cost ~0.7 ms of LSU / L2 sector work
    // at cfg4a)
    uint8_t* sOut = smem + L::kOutOff + warp * 4096;
    const int lr = static_cast<int>(lane_id());
    auto out_chunk = [&](int g) {
      return reinterpret_cast<uint4*>(sOut + lr * 128 + ((g ^ (lr & 7)) << 4));
    };
    SC_T0();
    for (int n = 0; n < nq; ++n) {
      const int t = n % kSS;
      const int q0 = (q_tiles - 1 - n) * 128;
      const int ib = q0 + half * 64;  // first query column of this warp
      // kept(i = ib + c, j) as one column range per thread: c in [c_lo, c_hi) (the band's lower
      // and upper query bounds for this key row; an out-of-range key keeps nothing)
      int c_lo = p.mask.causal ? j - p.mask.diag_offset - ib : INT_MIN / 2;
      int c_hi = p.mask.window > 0 ? j - p.mask.diag_offset + p.mask.window - ib : INT_MAX / 2;
      if (j >= p.seq_k) c_lo = INT_MAX / 2;
      const float* l2s = sStat + t * 256 + half * 64;
      const float* dls = l2s + 128;
      if (warp == 0 && lane_id() == 0) {
        SC_ACC(5, mbar_wait(&stat_full[t], (n / kSS) & 1));
        SC_ACC(6, mbar_wait(s_full, n & 1));
      }
      __syncwarp();
      mbar_wait(&stat_full[t], (n / kSS) & 1);
      mbar_wait(s_full, n & 1);
      tc_fence_after();
      uint32_t pr[64];  // S^T row, then P^T (fp32 bits)
      tmem_ld32(tmem + lane_base + kColS + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&pr[0]));
      tmem_ld32(tmem + lane_base + kColS + half * 64 + 32,
                *reinterpret_cast<uint32_t(*)[32]>(&pr[32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) {  // S^T read (tcgen05.wait::ld returned): the pair's MMA may reuse it
        if (leader)
          mbar_arrive(s_free);
        else
          mbar_arrive_cluster_relaxed(s_free_l);
      }
      {
        uint32_t pw[32];
#pragma unroll
        for (int e = 0; e < 64; e += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(l2s + e);
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const bool keep = (e + x >= c_lo) & (e + x < c_hi);
            // ex2(-inf) = 0: masked scores without a branch around the MUFU op
            const float pe = ex2(keep ? fmaf(__uint_as_float(pr[e + x]), p.scale_log2, -lv[x])
                                      : -INFINITY);
            pr[e + x] = __float_as_uint(pe);
          }
          pw[e / 2] = pack_bf16(__uint_as_float(pr[e]), __uint_as_float(pr[e + 1]));
          pw[e / 2 + 1] = pack_bf16(__uint_as_float(pr[e + 2]), __uint_as_float(pr[e + 3]));
        }
        if (lr == 0) bulk_wait_read<0>();  // the previous dS'^T store has read the box
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *out_chunk(v) = make_uint4(pw[v * 4], pw[v * 4 + 1], pw[v * 4 + 2], pw[v * 4 + 3]);
        fence_proxy_async_smem();
        __syncwarp();
#ifndef AF_SCORES_NO_STORE  // developer ablation (results are wrong without the stores)
        if (lr == 0) {
          tma_store_4d(&tm_pst, sOut, ib, k0 + wq * 32, bh, 0);
          bulk_commit();
        }
#endif
      }
      if (warp == 0 && lane_id() == 0) SC_ACC(7, mbar_wait(dp_full, n & 1));
      __syncwarp();
      mbar_wait(dp_full, n & 1);
      tc_fence_after();
#pragma unroll  // (P^T is indexed by hf: a rolled loop would put it in local memory)
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t dr[32];
        tmem_ld32(tmem + lane_base + kColDP + half * 64 + hf * 32, dr);
        tmem_ld_wait();
        if (hf == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) {
            if (leader)
              mbar_arrive(dp_free);
            else
              mbar_arrive_cluster_relaxed(dp_free_l);
          }
        }
        uint32_t dw[16];
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 d4 = *reinterpret_cast<const float4*>(dls + hf * 32 + e);
          const float dl[4] = {d4.x, d4.y, d4.z, d4.w};
          float dv[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const bool keep = (hf * 32 + e + x >= c_lo) & (hf * 32 + e + x < c_hi);
            // dS' is selected (not multiplied by P's zero): dP of a masked position need not be
            // finite
            dv[x] = keep ? __uint_as_float(pr[hf * 32 + e + x]) *
                               (__uint_as_float(dr[e + x]) - dl[x]) * sc
                         : 0.0f;
          }
          dw[e / 2] = pack_bf16(dv[0], dv[1]);
          dw[e / 2 + 1] = pack_bf16(dv[2], dv[3]);
        }
        if (hf == 0) {
          if (lr == 0) bulk_wait_read<0>();  // the P^T store has read the box
          __syncwarp();
        }
#pragma unroll
        for (int v = 0; v < 4; ++v)
          *out_chunk(hf * 4 + v) = make_uint4(dw[v * 4], dw[v * 4 + 1], dw[v * 4 + 2], dw[v * 4 + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
#ifndef AF_SCORES_NO_STORE
      if (lr == 0) {
        tma_store_4d(&tm_dsst, sOut, ib, k0 + wq * 32, bh, 0);
        bulk_commit();
      }
#endif
      // the statistics slot is released after its values have been consumed (an arrive right
      // after the shared loads does not wait for them, and the producer's next bulk copy into
      // the slot could land first)
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&stat_empty[t]);
    }
    if (lr == 0) bulk_wait<0>();
  }

  tc_fence_before();
  cluster_sync();  // the leader's last commits land in the peer's barriers before it exits
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
}

// ═══════════════════════════════ 2/3. dQ and key-side GEMMs ═══════════════════════════════
// One accumulator tile of 128 rows x N columns in TMEM, fed by a ring of stages:
//   stage = A (16 KB: one [128][64] K-major box, or two [64][64] boxes MN-major)
//         + B (N/64 boxes [64 K-rows][64 cols], MN-major)
// The scores are stored transposed, [B*H, k_pad, q_pad] (the scores kernel writes key rows):
// kGemmDQ : rows = queries of (b, h, q tile); items = visible key tiles; A = dS' (MN-major from
//           the key-row layout), B = K[hk][:, n0:n0+N].
// key side: rows = keys of (b, hk, key tile); items = (h in the head chunk, visible q tile); per
//           64-query chunk one or two products: A = dS'^T (K-major), B = Q[:, n0:] (dK, and MLA's
//           latent dKV) and A = P^T, B = dO[:, n0:] (dV, and MLA's dKV for n0 < 512).
enum GemmMode : int { kGemmDQ = 0, kGemmDKV = 1, kGemmDK = 2, kGemmDV = 3 };

template <int N>
struct MlaGemmSmem {
  static constexpr int kStages = N >= 256 ? 2 : 4;
  static constexpr int kABytes = 16384;
  static constexpr int kBBytes = (N / 64) * 8192;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kBarOff = kStages * kStage;
  static constexpr int kNumBars = 2 * kStages + 1;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
  static constexpr int kTmemCols = N > 256 ? 512 : (N > 128 ? 256 : (N > 64 ? 128 : 64));
};

template <int kMode, int N>
__global__ void __launch_bounds__(192, 1)
    mla_bwd_gemm_kernel(const __grid_constant__ CUtensorMap tm_a1,   // dS'
                        const __grid_constant__ CUtensorMap tm_a2,   // P (key side)
                        const __grid_constant__ CUtensorMap tm_b1,   // K (dQ) / Q (key side)
                        const __grid_constant__ CUtensorMap tm_b2,   // dO (key side)
                        const MlaBwdParams p, int n0) {
  using L = MlaGemmSmem<N>;
  constexpr int kStages = L::kStages;
  constexpr bool kKey = kMode != kGemmDQ;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);
  const int warp = static_cast<int>(warp_id());
  const int group = p.heads / p.heads_kv;

  // ── work decomposition ──
  int b, hk, tile, h_lo = 0, h_hi = 0, bh = 0, g = 0, bk = 0;
  int it_lo = 0, it_hi = 0;  // contraction tile range (key tiles for dQ, q tiles key-side)
  const int q_tiles = p.q_pad / 128;
  if constexpr (!kKey) {
    // blockIdx.x = (q tile, b*H + h), heaviest (last) query tiles first under a causal mask
    const int bhs = p.batch * p.heads;
    const int raw = static_cast<int>(blockIdx.x) / bhs;
    bh = static_cast<int>(blockIdx.x) % bhs;
    b = bh / p.heads;
    hk = (bh % p.heads) / group;
    tile = p.mask.causal ? q_tiles - 1 - raw : raw;
    const TileBand band = key_band(p.mask, tile * 128, min(p.seq_q, tile * 128 + 128), p.seq_k);
    it_lo = band.jb_lo;
    it_hi = band.jb_hi;
  } else {
    // blockIdx.x = (key tile, b*Hkv + hk, head chunk), heaviest (first) key tiles first
    const int per = p.batch * p.heads_kv * p.groups;
    tile = static_cast<int>(blockIdx.x) / per;
    const int rest = static_cast<int>(blockIdx.x) % per;
    bk = rest / p.groups;
    g = rest % p.groups;
    b = bk / p.heads_kv;
    hk = bk % p.heads_kv;
    h_lo = hk * group + g * group / p.groups;
    h_hi = hk * group + (g + 1) * group / p.groups;
    it_lo = mla_q_tile_lo(p.mask, tile * 128);
    it_hi = q_tiles;
  }
  // stages per contraction tile: two 64-row chunks x products
  const int per_item = (kMode == kGemmDKV && n0 < kMbDv) ? 4 : 2;
  const int n_items = kKey ? (h_hi - h_lo) * max(0, it_hi - it_lo) : max(0, it_hi - it_lo);
  const int n_stages_total = n_items * per_item;

  if (warp == 4 && lane_id() == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ───────────── TMA producer ─────────────
    if (elect_one()) {
      int slot = 0;
      uint32_t ph = 0;
      for (int st = 0; st < n_stages_total; ++st) {
        const int item = st / per_item, sub = st % per_item;
        mbar_wait(&empty[slot], ph ^ 1);
        mbar_expect_tx(&full[slot], L::kStage);
        uint8_t* sa = smem + slot * L::kStage;
        uint8_t* sb = sa + L::kABytes;
        if constexpr (!kKey) {
          const int kt = it_lo + item;
          const int c = sub;  // 64-key chunk
          // dS'^T rows [kt*128 + 64c, +64) x query columns of this tile: A MN-major, two boxes
          tma_load_4d(sa, &tm_a1, &full[slot], tile * 128, kt * 128 + c * 64, bh, 0);
          tma_load_4d(sa + 8192, &tm_a1, &full[slot], tile * 128 + 64, kt * 128 + c * 64, bh, 0);
          for (int nb = 0; nb < N / 64; ++nb)
            tma_load_4d_hint(sb + nb * 8192, &tm_b1, &full[slot], n0 + nb * 64,
                             kt * 128 + c * 64, hk, b, kEvictLast);
        } else {
          // query tiles from the last one down, the heads of the chunk inside each: the CTAs of
          // every key tile start at the last query tile and step down at the same pace (a key
          // tile just stops earlier), so they stream the same (q tile, head) Q / dO tile at the
          // same time and it is read from HBM once (head-outer, the CTAs drifted apart after the
          // first head — their per-head lengths differ — and re-read Q / dO ~10x from HBM)
          const int nh = h_hi - h_lo;
          const int qt = it_hi - 1 - item / nh;
          const int hh = h_lo + item % nh;
          // chunk, product (0: dS'/Q, 1: P/dO)
          const int c = per_item == 4 ? sub / 2 : sub;
          const int prod = per_item == 4 ? sub % 2 : (kMode == kGemmDV ? 1 : 0);
          const int bhh = b * p.heads + hh;
          const int r0 = qt * 128 + c * 64;
          const CUtensorMap* ta = prod == 0 ? &tm_a1 : &tm_a2;
          const CUtensorMap* tb = prod == 0 ? &tm_b1 : &tm_b2;
          // dS'^T / P^T rows of this key tile x 64 query columns: A K-major, one box
          tma_load_4d(sa, ta, &full[slot], r0, tile * 128, bhh, 0);
          for (int nb = 0; nb < N / 64; ++nb)
            tma_load_4d(sb + nb * 8192, tb, &full[slot], n0 + nb * 64, r0, hh, b);
        }
        if (++slot == kStages) {
          slot = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 5) {
    // ───────────── MMA issuer ─────────────
    if (elect_one()) {
      constexpr int kN = N >= 256 ? 256 : N;  // per-instruction N
      constexpr uint32_t id = make_idesc_bf16(128, kN, !kKey, true);
      int slot = 0;
      uint32_t ph = 0;
      for (int st = 0; st < n_stages_total; ++st) {
        mbar_wait(&full[slot], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + slot * L::kStage);
        const uint32_t sb = sa + L::kABytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = kKey ? make_sdesc(sa + kk * 32, 0, 1024)
                                   : make_sdesc(sa + kk * 2048, 8192, 1024);
#pragma unroll
          for (int nh = 0; nh < N / kN; ++nh)
            mma_ss(tmem + nh * kN, ad,
                   make_sdesc(sb + nh * (kN / 64) * 8192 + kk * 2048, 8192, 1024), id,
                   (st > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&empty[slot]);
        if (++slot == kStages) {
          slot = 0;
          ph ^= 1;
        }
      }
      mma_commit(acc_full);
    }
  } else {
    // ───────────── epilogue warps 0-3: one accumulator row per thread ─────────────
    const int row = warp * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    if (n_stages_total > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
    }
#pragma unroll 1
    for (int c = 0; c < N / 32; ++c) {
      uint32_t r[32];
      if (n_stages_total > 0) {
        tmem_ld32(tmem + lane_base + c * 32, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) r[e] = 0u;
      }
      if constexpr (!kKey) {
        const int i = tile * 128 + row;
        if (i < p.seq_q) {
          const int h = bh % p.heads;
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.dq) + b * p.dq_sb +
                               h * p.dq_sh + static_cast<int64_t>(i) * p.dq_ss + n0 + c * 32;
          uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            d4[v] = make_uint4(pack_bf16(__uint_as_float(r[v * 8]), __uint_as_float(r[v * 8 + 1])),
                               pack_bf16(__uint_as_float(r[v * 8 + 2]), __uint_as_float(r[v * 8 + 3])),
                               pack_bf16(__uint_as_float(r[v * 8 + 4]), __uint_as_float(r[v * 8 + 5])),
                               pack_bf16(__uint_as_float(r[v * 8 + 6]), __uint_as_float(r[v * 8 + 7])));
        }
      } else {
        const int j = tile * 128 + row;
        float* dst = p.dkv_part +
                     ((static_cast<int64_t>(g) * p.batch * p.heads_kv + bk) * p.k_pad + j) *
                         p.part_width +
                     n0 + c * 32;
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          d4[v] = make_float4(__uint_as_float(r[v * 4]), __uint_as_float(r[v * 4 + 1]),
                              __uint_as_float(r[v * 4 + 2]), __uint_as_float(r[v * 4 + 3]));
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<L::kTmemCols>(tmem);
  }
}

// ── the same GEMMs on a CTA pair (N = 128, 256, 512) ──
// M = 256 tcgen05.mma.cta_group::2: the pair's two row tiles (query tiles 2p, 2p+1 for dQ; key
// tiles 2p, 2p+1 key-side) are the A rows, each CTA loading its own; B (K / Q / dO columns) is
// split by N, each CTA loading half of every instruction's 256 (or N) columns — so every B byte is
// fetched from L2 once per two row tiles (the single-CTA GEMMs re-streamed B per row tile and were
// L2-throughput bound).  The pair walks the union of its tiles' contraction ranges; the extra
// causal block (key tile 2p+1 x query tile 2p) is the zero block the scores kernel writes.
template <int N>
struct MlaPairGemmSmem {
  static constexpr int kNI = N > 256 ? 256 : N;        // N per instruction
  static constexpr int kHalfBoxes = kNI / 2 / 64;      // this CTA's 64-col B blocks per instr.
  static constexpr int kABytes = 16384;
  static constexpr int kBBytes = (N / kNI) * kHalfBoxes * 8192;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kStagesFit = (224 * 1024) / kStage;
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  static constexpr int kBarOff = kStages * kStage;
  static constexpr int kNumBars = 2 * kStages + 1;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
  static constexpr int kTmemCols = N > 256 ? 512 : (N > 128 ? 256 : 128);
  static_assert(kNI % 128 == 0, "each CTA's half of an instruction's N is whole 64-col blocks");
  static_assert(4 * (N / 64) * 4096 <= kStages * kStage, "dQ staging fits the drained ring");
  static_assert(4 * 8 * 4096 <= kStages * kStage, "partial staging (one column half) fits");
};

template <int kMode, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    mla_bwd_gemm_pair_kernel(const __grid_constant__ CUtensorMap tm_a1,   // dS'
                             const __grid_constant__ CUtensorMap tm_a2,   // P (key side)
                             const __grid_constant__ CUtensorMap tm_b1,   // K (dQ) / Q (key side)
                             const __grid_constant__ CUtensorMap tm_b2,   // dO (key side)
                             const __grid_constant__ CUtensorMap tm_out,  // dQ / partials store
                             const MlaBwdParams p, int n0) {
  using L = MlaPairGemmSmem<N>;
  constexpr int kStages = L::kStages, kNI = L::kNI, kHB = L::kHalfBoxes;
  constexpr bool kKey = kMode != kGemmDQ;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);
  const int warp = static_cast<int>(warp_id());
  const int group = p.heads / p.heads_kv;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pairx = static_cast<int>(blockIdx.x) / 2;

  // ── work decomposition (per pair; the rank picks the row tile) ──
  int b, hk, tile, h_lo = 0, h_hi = 0, bh = 0, g = 0, bk = 0;
  int it_lo = 0, it_hi = 0;  // contraction tile range (key tiles for dQ, q tiles key-side)
  const int q_tiles = p.q_pad / 128;
  if constexpr (!kKey) {
    // pair = (q tile pair, b*H + h), heaviest (last) query tiles first under a causal mask
    const int bhs = p.batch * p.heads;
    const int raw = pairx / bhs;
    bh = pairx % bhs;
    b = bh / p.heads;
    hk = (bh % p.heads) / group;
    const int t0 = p.mask.causal ? q_tiles - 2 - 2 * raw : 2 * raw;
    tile = t0 + static_cast<int>(rank);
    const TileBand band = key_band(p.mask, t0 * 128, min(p.seq_q, t0 * 128 + 256), p.seq_k);
    it_lo = band.jb_lo;
    it_hi = band.jb_hi;
  } else {
    // pair = (key tile pair, b*Hkv + hk, head chunk), heaviest (first) key tiles first
    const int per = p.batch * p.heads_kv * p.groups;
    const int tp = pairx / per;
    const int rest = pairx % per;
    tile = 2 * tp + static_cast<int>(rank);
    bk = rest / p.groups;
    g = rest % p.groups;
    b = bk / p.heads_kv;
    hk = bk % p.heads_kv;
    h_lo = hk * group + g * group / p.groups;
    h_hi = hk * group + (g + 1) * group / p.groups;
    it_lo = mla_q_tile_lo(p.mask, 2 * tp * 128);
    it_hi = q_tiles;
  }
  const int per_item = (kMode == kGemmDKV && n0 < kMbDv) ? 4 : 2;
  const int n_items = kKey ? (h_hi - h_lo) * max(0, it_hi - it_lo) : max(0, it_hi - it_lo);
  const int n_stages_total = n_items * per_item;

  if (warp == 4 && lane_id() == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc_pair<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ───────────── TMA producer (each CTA: its A rows, its half of B) ─────────────
    if (elect_one()) {
      int slot = 0;
      uint32_t ph = 0;
      for (int st = 0; st < n_stages_total; ++st) {
        const int item = st / per_item, sub = st % per_item;
        mbar_wait(&empty[slot], ph ^ 1);
        if (leader) mbar_expect_tx(&full[slot], 2 * L::kStage);
        const uint32_t fl = peer_addr(&full[slot], 0);
        uint8_t* sa = smem + slot * L::kStage;
        uint8_t* sb = sa + L::kABytes;
        const CUtensorMap* tb;
        int brow, bc2, bc3;  // B tile coordinates: rows (contraction), head, batch
        if constexpr (!kKey) {
          const int kt = it_lo + item;
          const int c = sub;  // 64-key chunk
          // dS'^T rows [kt*128 + 64c, +64) x this CTA's query tile: A MN-major, two boxes
          tma_load_4d_pair(sa, &tm_a1, fl, tile * 128, kt * 128 + c * 64, bh, 0);
          tma_load_4d_pair(sa + 8192, &tm_a1, fl, tile * 128 + 64, kt * 128 + c * 64, bh, 0);
          tb = &tm_b1;
          brow = kt * 128 + c * 64;
          bc2 = hk;
          bc3 = b;
        } else {
          // query tiles from the last one down, the heads of the chunk inside each (the CTAs of
          // every key tile pair stream the same (q tile, head) tile at the same time)
          const int nh = h_hi - h_lo;
          const int qt = it_hi - 1 - item / nh;
          const int hh = h_lo + item % nh;
          const int c = per_item == 4 ? sub / 2 : sub;
          const int prod = per_item == 4 ? sub % 2 : (kMode == kGemmDV ? 1 : 0);
          const int r0 = qt * 128 + c * 64;
          // dS'^T / P^T rows of this CTA's key tile x 64 query columns: A K-major, one box
          tma_load_4d_pair(sa, prod == 0 ? &tm_a1 : &tm_a2, fl, r0, tile * 128,
                           b * p.heads + hh, 0);
          tb = prod == 0 ? &tm_b1 : &tm_b2;
          brow = r0;
          bc2 = hh;
          bc3 = b;
        }
        // this CTA's half of each instruction's kNI columns: [nh*kNI + rank*kNI/2, +kNI/2)
#pragma unroll
        for (int nh = 0; nh < N / kNI; ++nh)
#pragma unroll
          for (int x = 0; x < kHB; ++x)
            tma_load_4d_pair(sb + (nh * kHB + x) * 8192, tb, fl,
                             n0 + nh * kNI + static_cast<int>(rank) * (kNI / 2) + x * 64, brow,
                             bc2, bc3);
        if (++slot == kStages) {
          slot = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 5) {
    // ───────────── MMA issuer (the leader, for both CTAs) ─────────────
    if (leader && n_stages_total > 0 && elect_one()) {
      constexpr uint32_t id = make_idesc_bf16(256, kNI, !kKey, true);
      int slot = 0;
      uint32_t ph = 0;
      for (int st = 0; st < n_stages_total; ++st) {
        mbar_wait(&full[slot], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + slot * L::kStage);
        const uint32_t sb = sa + L::kABytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = kKey ? make_sdesc(sa + kk * 32, 0, 1024)
                                   : make_sdesc(sa + kk * 2048, 8192, 1024);
#pragma unroll
          for (int nh = 0; nh < N / kNI; ++nh)
            mma_ss_pair(tmem + nh * kNI, ad, make_sdesc(sb + nh * kHB * 8192 + kk * 2048, 8192, 1024),
                        id, (st > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit_pair(&empty[slot]);
        if (++slot == kStages) {
          slot = 0;
          ph ^= 1;
        }
      }
      mma_commit_pair(acc_full);
    }
  } else {
    // ───────────── epilogue warps 0-3: one accumulator row per thread (this CTA's rows) ─────────────
    const int row = warp * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    if (n_stages_total > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
    }
#pragma unroll 1
    for (int c = 0; c < N / 32; ++c) {
      uint32_t r[32];
      if (n_stages_total > 0) {
        tmem_ld32(tmem + lane_base + c * 32, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) r[e] = 0u;
      }
      if constexpr (!kKey) {
        const int i = tile * 128 + row;
        if (p.dq_tma) {  // this warp's rows into its 64-column boxes of the drained ring
          uint8_t* bx = smem + (warp * (N / 64) + c / 2) * 4096;
          const int lr = static_cast<int>(lane_id());
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int gq = (c % 2) * 4 + v;
            *reinterpret_cast<uint4*>(bx + lr * 128 + ((gq ^ (lr & 7)) << 4)) =
                make_uint4(pack_bf16(__uint_as_float(r[v * 8]), __uint_as_float(r[v * 8 + 1])),
                           pack_bf16(__uint_as_float(r[v * 8 + 2]), __uint_as_float(r[v * 8 + 3])),
                           pack_bf16(__uint_as_float(r[v * 8 + 4]), __uint_as_float(r[v * 8 + 5])),
                           pack_bf16(__uint_as_float(r[v * 8 + 6]), __uint_as_float(r[v * 8 + 7])));
          }
        } else if (i < p.seq_q) {
          const int h = bh % p.heads;
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.dq) + b * p.dq_sb +
                               h * p.dq_sh + static_cast<int64_t>(i) * p.dq_ss + n0 + c * 32;
          uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            d4[v] = make_uint4(pack_bf16(__uint_as_float(r[v * 8]), __uint_as_float(r[v * 8 + 1])),
                               pack_bf16(__uint_as_float(r[v * 8 + 2]), __uint_as_float(r[v * 8 + 3])),
                               pack_bf16(__uint_as_float(r[v * 8 + 4]), __uint_as_float(r[v * 8 + 5])),
                               pack_bf16(__uint_as_float(r[v * 8 + 6]), __uint_as_float(r[v * 8 + 7])));
        }
      } else if (p.part_tma) {
        // fp32 partial rows into [32 rows][32 cols] SW128 boxes of the drained ring, in two
        // column halves (256 columns = 8 boxes per warp per half)
        const int hc = c / 8;  // column half of N = 512 (c counts 32-column chunks)
        if (c % 8 == 0 && hc > 0) {  // the first half's stores have read the boxes
          if (lane_id() == 0) bulk_wait_read<0>();
          __syncwarp();
        }
        uint8_t* bx = smem + (warp * 8 + c % 8) * 4096;
        const int lr = static_cast<int>(lane_id());
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<float4*>(bx + lr * 128 + ((v ^ (lr & 7)) << 4)) =
              make_float4(__uint_as_float(r[v * 4]), __uint_as_float(r[v * 4 + 1]),
                          __uint_as_float(r[v * 4 + 2]), __uint_as_float(r[v * 4 + 3]));
        if (c % 8 == 7 || c == N / 32 - 1) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane_id() == 0) {
            for (int x = 0; x <= c % 8; ++x)
              tma_store_4d(&tm_out, smem + (warp * 8 + x) * 4096, n0 + (hc * 8 + x) * 32,
                           tile * 128 + warp * 32, bk, g);
            bulk_commit();
          }
        }
      } else {
        const int j = tile * 128 + row;
        float* dst = p.dkv_part +
                     ((static_cast<int64_t>(g) * p.batch * p.heads_kv + bk) * p.k_pad + j) *
                         p.part_width +
                     n0 + c * 32;
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          d4[v] = make_float4(__uint_as_float(r[v * 4]), __uint_as_float(r[v * 4 + 1]),
                              __uint_as_float(r[v * 4 + 2]), __uint_as_float(r[v * 4 + 3]));
      }
    }
    if constexpr (kKey) {
      if (p.part_tma && lane_id() == 0) bulk_wait<0>();
    }
    if constexpr (!kKey) {
      if (p.dq_tma) {  // N / 64 boxes of [32 rows][64 cols]; rows past seq_q are clipped
        fence_proxy_async_smem();
        __syncwarp();
        if (lane_id() == 0) {
          const int h = bh % p.heads;
          for (int x = 0; x < N / 64; ++x)
            tma_store_4d(&tm_out, smem + (warp * (N / 64) + x) * 4096, n0 + x * 64,
                         tile * 128 + warp * 32, h, b);
          bulk_commit();
          bulk_wait<0>();
        }
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc_pair<L::kTmemCols>(tmem);
  }
}

// out[b, hk, j, :] = bf16( sum_g part[g, b*Hkv + hk, j, :] )  (group order fixed: deterministic)
__global__ void mla_bwd_reduce_kernel(const float* __restrict__ part, int groups, int bhk,
                                      int heads_kv, int seq_k, int k_pad, int width, int pitch,
                                      __nv_bfloat16* __restrict__ out, int64_t o_sb,
                                      int64_t o_sh, int64_t o_ss) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // 4 cols
  const int64_t per_row = width / 4;
  const int64_t total = static_cast<int64_t>(bhk) * seq_k * per_row;
  if (idx >= total) return;
  const int c4 = static_cast<int>(idx % per_row);
  const int64_t bj = idx / per_row;
  const int bk = static_cast<int>(bj / seq_k), j = static_cast<int>(bj % seq_k);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int g = 0; g < groups; ++g) {
    const float4 v = *reinterpret_cast<const float4*>(
        part + ((static_cast<int64_t>(g) * bhk + bk) * k_pad + j) * pitch + c4 * 4);
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  const int b = bk / heads_kv, hk = bk % heads_kv;
  *reinterpret_cast<uint2*>(out + b * o_sb + hk * o_sh + static_cast<int64_t>(j) * o_ss +
                            c4 * 4) = make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
}

}  // namespace af
