// K1t — softmax forward with one 128-row query tile per CTA and P in its own TMEM columns.
//
// In K1 (parallel_fwd.cuh) two query tiles ping-pong and P is packed into the columns of the S
// it came from, so S(n+1) of a tile cannot be computed before PV(n) has read P(n): the per-tile
// period is softmax + PV + S (tools/trace_fwd.py).  Here one tile owns
//   TMEM: S0 [0,128) | S1 [128,256) | P0 [256,320) | P1 [320,384) | O [384, 384+DV)
// so S(n+2) is issued as soon as the row warps have loaded S(n) into registers, and the softmax of
// block n+1 no longer waits for PV(n): the period becomes max(softmax, S + PV).  The price is
// twice the K/V L2 -> SMEM traffic (a K/V tile serves 128 query rows instead of 256).
// Warps: 0-7 softmax rows (two per row, 64 key columns each, block max exchanged per block;
// lazy rescale, packed FFMA2/FADD2, 1/8 of the exponentials as a polynomial), 8 TMA, 9 MMA.
#pragma once
#include "parallel_fwd.cuh"

namespace af {

template <int D, int DV>
struct Fwd1tSmem {
  static constexpr int kStages = D == 128 ? 3 : 4;
  static constexpr int kQBytes = kBlockM * D * 2;
  static constexpr int kKBytes = kBlockN * D * 2;
  static constexpr int kVBytes = kBlockN * DV * 2;
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + kQBytes;
  static constexpr int kVOff = kKOff + kStages * kKBytes;
  static constexpr int kBarOff = kVOff + kStages * kVBytes;
  // q_full, k_full[S], k_empty[S], v_full[S], v_empty[S], s_full[2], s_free[2], p_full[2],
  // p_free[2]
  static constexpr int kNumBars = 1 + 4 * kStages + 8;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  // block-max exchange [2 slots][2 halves][128]; the final row sums reuse slot nk % 2
  static constexpr int kRowMaxOff = kTmemSlotOff + 16;
  static constexpr int kTotal = kRowMaxOff + 2 * 2 * 128 * 4;
};
constexpr int kFwd1tThreads = 320;  // 8 row warps (two per row), TMA warp 8, MMA warp 9

template <int D, int DV>
__global__ void __launch_bounds__(kFwd1tThreads, 1)
    parallel_fwd_1t_kernel(const __grid_constant__ CUtensorMap tm_q,
                           const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const ParallelFwdParams p) {
  using L = Fwd1tSmem<D, DV>;
  constexpr int kSt = L::kStages;
  static_assert(D % 64 == 0 && DV % 64 == 0 && D <= 128 && DV <= 128, "tile dims");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + kSt;
  uint64_t* v_full = k_empty + kSt;
  uint64_t* v_empty = v_full + kSt;
  uint64_t* s_full = v_empty + kSt;  // [2] S(n) in S_{n%2}
  uint64_t* s_free = s_full + 2;     // [2] the rows have S(n) in registers
  uint64_t* p_full = s_free + 2;     // [2] P(n) in P_{n%2}
  uint64_t* p_free = p_full + 2;     // [2] PV(n) done (P_{n%2} free; O holds blocks <= n)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);
  float* sRowMax = reinterpret_cast<float*>(smem + L::kRowMaxOff);

  const int warp = static_cast<int>(warp_id());
  const int q_tiles = (p.seq_q + kBlockM - 1) / kBlockM;
  const int qt = p.mask.causal ? (q_tiles - 1 - static_cast<int>(blockIdx.x))
                               : static_cast<int>(blockIdx.x);
  const int bh = blockIdx.y;
  const int b = bh / p.heads_q;
  const int h = bh % p.heads_q;
  const int hk = h / (p.heads_q / p.heads_kv);
  const int q0 = qt * kBlockM;
  const TileBand band = key_band(p.mask, q0, min(p.seq_q, q0 + kBlockM), p.seq_k);
  const int nk = band.jb_hi - band.jb_lo;

  if (warp == 8 && lane_id() == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&s_free[x], 8);
      mbar_init(&p_full[x], 8);
      mbar_init(&p_free[x], 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kColS = 0, kColP = 256, kColO = 384;

  if (warp == 8) {
    // ───────────── TMA producer ─────────────
    if (elect_one() && nk > 0) {
      mbar_expect_tx(q_full, L::kQBytes);
      for (int c = 0; c < D / 64; ++c)
        tma_load_4d(sQ + c * (kBlockM * 128), &tm_q, q_full, c * 64, q0, h, b);
      for (int n = 0; n < nk; ++n) {
        const int s = n % kSt;
        const uint32_t ph = (n / kSt) & 1;
        const int kv0 = (band.jb_lo + n) * kBlockN;
        mbar_wait(&k_empty[s], ph ^ 1);
        mbar_expect_tx(&k_full[s], L::kKBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d_hint(sK + s * L::kKBytes + c * (kBlockN * 128), &tm_k, &k_full[s], c * 64,
                           kv0, hk, b, kEvictLast);
        mbar_wait(&v_empty[s], ph ^ 1);
        mbar_expect_tx(&v_full[s], L::kVBytes);
        for (int c = 0; c < DV / 64; ++c)
          tma_load_4d_hint(sV + s * L::kVBytes + c * (kBlockN * 128), &tm_v, &v_full[s], c * 64,
                           kv0, hk, b, kEvictLast);
      }
    }
  } else if (warp == 9) {
    // ───────────── MMA issuer ─────────────
    if (elect_one() && nk > 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(kBlockM, kBlockN, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(kBlockM, DV, false, true);
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV);
      auto issue_s = [&](int n) {
        const int s = n % kSt;
        mbar_wait(&k_full[s], (n / kSt) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * (kBlockM * 128) + (kk % 4) * 32;
          mma_ss(tmem + kColS + (n & 1) * kBlockN, make_sdesc(aQ + off, 0, 1024),
                 make_sdesc(aK + s * L::kKBytes + (kk / 4) * (kBlockN * 128) + (kk % 4) * 32, 0,
                            1024),
                 idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[n & 1]);
        mma_commit(&k_empty[s]);  // K(n): read only by S(n)
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      issue_s(0);
      if (nk > 1) issue_s(1);
      for (int n = 0; n < nk; ++n) {
        const int x = n & 1;
        const int s = n % kSt;
        // S(n+2) into S_x as soon as the rows hold S(n) in registers
        if (n + 2 < nk) {
          mbar_wait(&s_free[x], (n >> 1) & 1);
          tc_fence_after();
          issue_s(n + 2);
        }
        AF_TRACE(8, n, 0);
        mbar_wait(&p_full[x], (n >> 1) & 1);
        AF_TRACE(8, n, 1);
        mbar_wait(&v_full[s], (n / kSt) & 1);
        AF_TRACE(8, n, 2);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kBlockN / 16; ++kk)
          mma_ts(tmem + kColO, tmem + kColP + x * (kBlockN / 2) + kk * 8,
                 make_sdesc(aV + s * L::kVBytes + kk * 16 * 128, kBlockN * 128, 1024), idesc_o,
                 (n > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&p_free[x]);
        mma_commit(&v_empty[s]);
      }
    }
  } else {
    // ───────────── softmax rows: two warps per row, 64 key columns each ─────────────
    const int wq = warp % 4;        // TMEM lane quarter
    const int ch = warp / 4;        // key-column half
    const int row = wq * 32 + static_cast<int>(lane_id());
    const int i = q0 + row;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t o_tmem = tmem + lane_base + kColO + ch * (DV / 2);
    const int pair_bar = 1 + wq;    // named barrier of the two warps sharing these rows
    float m_run = -INFINITY, l_run = 0.0f;
    for (int n = 0; n < nk; ++n) {
      const int x = n & 1;
      const int c0 = (band.jb_lo + n) * kBlockN;
      const int cb = c0 + ch * 64;
      mbar_wait(&s_full[x], (n >> 1) & 1);
      if (ch == 0) AF_TRACE(wq, n, 0);
      tc_fence_after();
      uint32_t sr[64];
      tmem_ld32(tmem + lane_base + kColS + x * kBlockN + ch * 64,
                *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      tmem_ld32(tmem + lane_base + kColS + x * kBlockN + ch * 64 + 32,
                *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&s_free[x]);  // S_x may take S(n+2)
      if (ch == 0) AF_TRACE(wq, n, 1);
      float* s = reinterpret_cast<float*>(sr);
      const bool full = block_fully_kept(p.mask, q0, c0, p.seq_k);
      const bool fast = full && p.scale_log2 > 0.0f;
      float bmax = -INFINITY;
      if (fast) {
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 64; c += 2)
          mx4[(c / 2) & 3] = fmaxf(mx4[(c / 2) & 3], fmaxf(s[c], s[c + 1]));
        bmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * p.scale_log2;
      } else {
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          s[c] = (full | kept(p.mask, i, cb + c, p.seq_k)) ? s[c] * p.scale_log2 : -INFINITY;
          bmax = fmaxf(bmax, s[c]);
        }
      }
      // block row max over both halves (slot n % 2: the partner's next write goes to the
      // other slot, and the one after follows its read of this one)
      float* mx = sRowMax + (n & 1) * 256;
      mx[ch * 128 + row] = bmax;
      named_bar_sync(pair_bar, 64);
      bmax = fmaxf(bmax, mx[(1 - ch) * 128 + row]);
      const float m_new = fmaxf(m_run, bmax);
      const bool need = (m_new - m_run) > 8.0f;  // lazy rescale (same decision in both halves)
      float factor = 1.0f;
      if (need) {
        factor = (m_run == -INFINITY) ? 0.0f : ex2(m_run - m_new);
        m_run = m_new;
      }
      const float m_use = (m_run == -INFINITY) ? 0.0f : m_run;
      if (ch == 0) AF_TRACE(wq, n, 2);
      uint32_t pk[32];
      float2 ls2[2] = {splat2(0.0f), splat2(0.0f)};
      if (fast) {
        const float2 sc2 = splat2(p.scale_log2), nm2 = splat2(-m_use);
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float2 xx = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
          const bool poly = (c & AF_EXP2_POLY_MASK) == 0;
          const float2 e = poly ? exp2_poly2(xx) : make_float2(ex2(xx.x), ex2(xx.y));
          ls2[(c / 2) & 1] = fadd2(ls2[(c / 2) & 1], e);
          pk[c / 2] = pack_bf16(e.x, e.y);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float2 e = make_float2(ex2(s[c] - m_use), ex2(s[c + 1] - m_use));
          ls2[(c / 2) & 1] = fadd2(ls2[(c / 2) & 1], e);
          pk[c / 2] = pack_bf16(e.x, e.y);
        }
      }
      l_run = l_run * factor + ((ls2[0].x + ls2[1].x) + (ls2[0].y + ls2[1].y));
      if (ch == 0) AF_TRACE(wq, n, 3);
      // O correction of this warp's columns (rows whose max moved by > 2^8): PV(n-1) in O
      if (n > 0 && __any_sync(0xffffffffu, need)) {
        mbar_wait(&p_free[(n - 1) & 1], ((n - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < DV / 64; ++c) {
          uint32_t orr[32];
          tmem_ld32(o_tmem + c * 32, orr);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) orr[e] = __float_as_uint(__uint_as_float(orr[e]) * factor);
          tmem_st32(o_tmem + c * 32, orr);
        }
        tmem_st_wait();
      }
      // P_x is free once PV(n-2) has read it; this half's 32 packed columns
      if (n >= 2) {
        mbar_wait(&p_free[x], ((n - 2) >> 1) & 1);
        tc_fence_after();
      }
      tmem_st32(tmem + lane_base + kColP + x * (kBlockN / 2) + ch * 32, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&p_full[x]);
      if (ch == 0) AF_TRACE(wq, n, 5);
    }
    // ───────────── epilogue: O / l (this warp's DV/2 columns), LSE ─────────────
    float* sRowSum = sRowMax + (nk & 1) * 256;  // last read two exchanges ago
    sRowSum[ch * 128 + row] = l_run;
    named_bar_sync(pair_bar, 64);
    const float total = sRowSum[row] + sRowSum[128 + row];
    const float inv = (total == 0.0f) ? 0.0f : 1.0f / total;
    if (nk > 0) {
      mbar_wait(&p_free[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
      tc_fence_after();
    }
    __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o) + b * p.o_stride_b +
                          h * p.o_stride_h +
                          static_cast<int64_t>(i < p.seq_q ? i : 0) * p.o_stride_s + ch * (DV / 2);
#pragma unroll
    for (int c = 0; c < DV / 64; ++c) {
      uint32_t orr[32];
      if (nk > 0) {
        tmem_ld32(o_tmem + c * 32, orr);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) orr[e] = 0u;
      }
      if (i < p.seq_q) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v)
          dst[v] = make_uint4(
              pack_bf16(__uint_as_float(orr[v * 8 + 0]) * inv, __uint_as_float(orr[v * 8 + 1]) * inv),
              pack_bf16(__uint_as_float(orr[v * 8 + 2]) * inv, __uint_as_float(orr[v * 8 + 3]) * inv),
              pack_bf16(__uint_as_float(orr[v * 8 + 4]) * inv, __uint_as_float(orr[v * 8 + 5]) * inv),
              pack_bf16(__uint_as_float(orr[v * 8 + 6]) * inv, __uint_as_float(orr[v * 8 + 7]) * inv));
      }
    }
    if (ch == 0 && p.lse != nullptr && i < p.seq_q)
      p.lse[(static_cast<int64_t>(b) * p.heads_q + h) * p.seq_q + i] =
          (total == 0.0f) ? -INFINITY : (m_run * kLn2 + logf(total));
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace af
