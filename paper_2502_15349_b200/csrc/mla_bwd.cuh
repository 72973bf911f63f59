// K3b — MLA backward on sm_100a (DeepSeek-V2 latent attention: Dqk = 576, Dv = 512, one KV head
// shared by every query head, V = K[:, :512]).
//
// The VJP is the softmax-family closed form of K2 with the latent aliasing of
// SURVEY §8c(1):  dKV = sum_h (tau dS_h^T Q_h) + [sum_h P_h^T dO_h, 0].
//
// Why not K2's fused key-/query-stationary kernels: a 128 x 576 fp32 accumulator (288 KB) does not
// fit in TMEM (256 KB), and a 128-row Q/dO tile pair is 272 KB of shared memory.  Instead the
// backward is split into dense tensor-core phases that each fit the SM:
//   1. scores   (key-tile stationary, K tile resident in smem, Q/dO streamed in 64-column boxes):
//               S = Q K^T, dP = dO V^T into double-buffered TMEM; row warps write
//               P = exp(S tau - LSE) and dS' = tau P (dP - D) as bf16 tiles to HBM (only the
//               causal blocks; padded rows/cols written as zeros).
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
};

// ═══════════════════════════════ 1. scores ═══════════════════════════════

template <int D, int DV, bool kShared>
struct MlaScoresSmem {
  static constexpr int kBox = 128 * 128;              // [128 rows][64 bf16]
  static constexpr int kKB = D / 64, kVB = DV / 64;   // boxes per K / V row tile
  // ring depth: whatever shared memory the resident K (and V) tile leaves (the streamed Q / dO
  // boxes are consumed in ~256 cycles each, so the ring depth sets the bytes in flight)
  static constexpr int kStages =
      (225 * 1024 - (kKB + (kShared ? 0 : kVB)) * kBox - 4096) / kBox > 12
          ? 12
          : (225 * 1024 - (kKB + (kShared ? 0 : kVB)) * kBox - 4096) / kBox;
  static constexpr int kKOff = 0;                     // the resident K (and V) tile
  static constexpr int kVOff = kKOff + kKB * kBox;
  static constexpr int kRingOff = kVOff + (kShared ? 0 : kVB) * kBox;  // streamed Q / dO boxes
  static constexpr int kStatOff = kRingOff + kStages * kBox;  // [2][2][128] fp32
  static constexpr int kBarOff = kStatOff + 2 * 2 * 128 * 4;
  // k_full, full[S], empty[S], stat_full[2], stat_empty[2], s_full[2], acc_empty[2]
  static constexpr int kNumBars = 1 + 2 * kStages + 8;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
};

__host__ __device__ inline int mla_q_tile_lo(const MaskParams& m, int k0) {
  // first 128-row query tile that sees key k0 under a top-left causal band
  return m.causal ? max(0, k0 - m.diag_offset) / 128 : 0;
}

template <int D, int DV, bool kShared>
__global__ void __launch_bounds__(320, 1)
    mla_bwd_scores_kernel(const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const MlaBwdParams p) {
  using L = MlaScoresSmem<D, DV, kShared>;
  constexpr int kStages = L::kStages;
  constexpr int kKB = L::kKB, kVB = L::kVB, kPerTile = kKB + kVB;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = kShared ? sK : smem + L::kVOff;
  uint8_t* sRing = smem + L::kRingOff;
  float* sStat = reinterpret_cast<float*>(smem + L::kStatOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* k_full = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + kStages;
  uint64_t* stat_full = empty + kStages;
  uint64_t* stat_empty = stat_full + 2;
  uint64_t* s_full = stat_empty + 2;
  uint64_t* acc_empty = s_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);

  const int warp = static_cast<int>(warp_id());
  // CTA order (b, h)-major with the key tiles of one head adjacent, and every CTA walks its query
  // tiles from the last one down: the CTAs of one head stream the same Q / dO tiles at the same
  // time, so each is read from HBM once and served to the other key tiles from L2.
  const int k_tiles = p.k_pad / 128;
  const int kt = static_cast<int>(blockIdx.x) % k_tiles;
  const int bh = static_cast<int>(blockIdx.x) / k_tiles;
  const int b = bh / p.heads, h = bh % p.heads;
  const int hk = h / (p.heads / p.heads_kv);
  const int k0 = kt * 128;
  const int q_tiles = p.q_pad / 128;
  const int qt_lo = mla_q_tile_lo(p.mask, k0);
  const int nq = q_tiles - qt_lo;

  if (warp == 8 && lane_id() == 0) {
    mbar_init(k_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&stat_full[t], 1);
      mbar_init(&stat_empty[t], 8);
      mbar_init(&s_full[t], 1);
      mbar_init(&acc_empty[t], 8);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ───────────── TMA producer ─────────────
    if (elect_one() && nq > 0) {
      mbar_expect_tx(k_full, (kKB + (kShared ? 0 : kVB)) * L::kBox);
      for (int c = 0; c < kKB; ++c) tma_load_4d(sK + c * L::kBox, &tm_k, k_full, c * 64, k0, hk, b);
      if constexpr (!kShared)
        for (int c = 0; c < kVB; ++c)
          tma_load_4d(sV + c * L::kBox, &tm_v, k_full, c * 64, k0, hk, b);
      int slot = 0;
      uint32_t ph = 0;
      for (int n = 0; n < nq; ++n) {
        const int q0 = (q_tiles - 1 - n) * 128;
        const int t = n & 1;
        mbar_wait(&stat_empty[t], ((n >> 1) & 1) ^ 1);
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
        for (int c = 0; c < kPerTile; ++c) {
          mbar_wait(&empty[slot], ph ^ 1);
          mbar_expect_tx(&full[slot], L::kBox);
          if (c < kKB)
            tma_load_4d(sRing + slot * L::kBox, &tm_q, &full[slot], c * 64, q0, h, b);
          else
            tma_load_4d(sRing + slot * L::kBox, &tm_do, &full[slot], (c - kKB) * 64, q0, h, b);
          if (++slot == kStages) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 9) {
    // ───────────── MMA issuer ─────────────
    if (elect_one() && nq > 0) {
      constexpr uint32_t id = make_idesc_bf16(128, 128, false, false);
      const uint32_t aR = smem_u32(sRing), aK = smem_u32(sK), aV = smem_u32(sV);
      mbar_wait(k_full, 0);
      int slot = 0;
      uint32_t ph = 0;
      for (int n = 0; n < nq; ++n) {
        const int t = n & 1;
        mbar_wait(&acc_empty[t], ((n >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_s = tmem + t * 256, d_dp = tmem + t * 256 + 128;
        for (int c = 0; c < kPerTile; ++c) {
          mbar_wait(&full[slot], ph);
          tc_fence_after();
          const bool is_s = c < kKB;
          // S += Q_c K_c^T ; dP += dO_c V_c^T (MLA: V = K boxes 0 .. Dv/64 - 1)
          const uint32_t bb = is_s ? aK + c * L::kBox : aV + (c - kKB) * L::kBox;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ss(is_s ? d_s : d_dp, make_sdesc(aR + slot * L::kBox + kk * 32, 0, 1024),
                   make_sdesc(bb + kk * 32, 0, 1024), id,
                   (c == 0 || c == kKB) && kk == 0 ? 0u : 1u);
          mma_commit(&empty[slot]);
          if (++slot == kStages) {
            slot = 0;
            ph ^= 1;
          }
        }
        mma_commit(&s_full[t]);
      }
    }
  } else {
    // ───────────── query-row warps: P and dS' rows ─────────────
    const int wq = warp % 4, half = warp / 4;
    const int row = wq * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const int cb = half * 64;
    for (int n = 0; n < nq; ++n) {
      const int t = n & 1;
      const int q0 = (q_tiles - 1 - n) * 128;
      const int i = q0 + row;
      mbar_wait(&stat_full[t], (n >> 1) & 1);
      const float l2 = sStat[t * 256 + row];
      const float dl = sStat[t * 256 + 128 + row];
      mbar_wait(&s_full[t], (n >> 1) & 1);
      tc_fence_after();
      // two 32-column halves (S and dP of one half live at a time: all 64 + 64 columns plus
      // the packed outputs at once needed ~190 registers and spilled at the 168 cap)
      const bool full_blk = block_fully_kept(p.mask, q0, k0, p.seq_k) && q0 + 128 <= p.seq_q;
      const int64_t off = (static_cast<int64_t>(bh) * p.q_pad + i) * p.k_pad + k0 + cb;
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t sr[32], dr[32];
        tmem_ld32(tmem + lane_base + t * 256 + cb + hf * 32, sr);
        tmem_ld32(tmem + lane_base + t * 256 + 128 + cb + hf * 32, dr);
        tmem_ld_wait();
        if (hf == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&acc_empty[t]);
        }
        uint32_t pw[16], dw[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float pv[2], dv[2];
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            const int j = k0 + cb + hf * 32 + e + x;
            const bool keep = full_blk | kept(p.mask, i, j, p.seq_k);
            // ex2(-inf) = 0: masked scores without a branch around the MUFU op; dS' is selected
            // (not multiplied by the zero) since dP of a masked position need not be finite
            const float pe =
                ex2(keep ? fmaf(__uint_as_float(sr[e + x]), p.scale_log2, -l2) : -INFINITY);
            pv[x] = pe;
            dv[x] = keep ? pe * (__uint_as_float(dr[e + x]) - dl) * p.scale : 0.0f;
          }
          pw[e / 2] = pack_bf16(pv[0], pv[1]);
          dw[e / 2] = pack_bf16(dv[0], dv[1]);
        }
        uint4* pd = reinterpret_cast<uint4*>(p.p + off + hf * 32);
        uint4* dd = reinterpret_cast<uint4*>(p.ds + off + hf * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          pd[v] = make_uint4(pw[v * 4], pw[v * 4 + 1], pw[v * 4 + 2], pw[v * 4 + 3]);
          dd[v] = make_uint4(dw[v * 4], dw[v * 4 + 1], dw[v * 4 + 2], dw[v * 4 + 3]);
        }
      }
      // release the statistics slot only after l2 / dl have been consumed (the stores above
      // depend on them): an arrive right after the shared loads does not wait for them to
      // return, and the producer's next bulk copy (async proxy) into this slot could land first
      // — measured at cfg4a as whole 32 x 64 P / dS' blocks computed with the LSE of tile n+2
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&stat_empty[t]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ═══════════════════════════════ 2/3. dQ and key-side GEMMs ═══════════════════════════════
// One accumulator tile of 128 rows x N columns in TMEM, fed by a ring of stages:
//   stage = A (16 KB: one [128][64] K-major box, or two [64][64] boxes MN-major)
//         + B (N/64 boxes [64 K-rows][64 cols], MN-major)
// kGemmDQ : rows = queries of (b, h, q tile); items = visible key tiles; A = dS' (K-major),
//           B = K[hk][:, n0:n0+N].
// key side: rows = keys of (b, hk, key tile); items = (h in the head chunk, visible q tile); per
//           64-query chunk one or two products: A = dS'^T (MN-major), B = Q[:, n0:] (dK, and MLA's
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
          tma_load_4d(sa, &tm_a1, &full[slot], kt * 128 + c * 64, tile * 128, bh, 0);
          for (int nb = 0; nb < N / 64; ++nb)
            tma_load_4d_hint(sb + nb * 8192, &tm_b1, &full[slot], n0 + nb * 64,
                             kt * 128 + c * 64, hk, b, kEvictLast);
        } else {
          // query tiles from the last one down: CTAs of different key tiles then stream the same
          // Q / dO tiles concurrently (L2 reuse)
          const int hh = h_lo + item / (it_hi - it_lo);
          const int qt = it_hi - 1 - item % (it_hi - it_lo);
          // chunk, product (0: dS'/Q, 1: P/dO)
          const int c = per_item == 4 ? sub / 2 : sub;
          const int prod = per_item == 4 ? sub % 2 : (kMode == kGemmDV ? 1 : 0);
          const int bhh = b * p.heads + hh;
          const int r0 = qt * 128 + c * 64;
          const CUtensorMap* ta = prod == 0 ? &tm_a1 : &tm_a2;
          const CUtensorMap* tb = prod == 0 ? &tm_b1 : &tm_b2;
          tma_load_4d(sa, ta, &full[slot], tile * 128, r0, bhh, 0);
          tma_load_4d(sa + 8192, ta, &full[slot], tile * 128 + 64, r0, bhh, 0);
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
      constexpr uint32_t id = make_idesc_bf16(128, kN, kKey, true);
      int slot = 0;
      uint32_t ph = 0;
      for (int st = 0; st < n_stages_total; ++st) {
        mbar_wait(&full[slot], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + slot * L::kStage);
        const uint32_t sb = sa + L::kABytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = kKey ? make_sdesc(sa + kk * 2048, 8192, 1024)
                                   : make_sdesc(sa + kk * 32, 0, 1024);
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
