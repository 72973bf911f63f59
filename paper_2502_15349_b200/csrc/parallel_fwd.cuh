// K1 — parallel-template forward on sm_100a.
//
// Replaces the arithmetic of attnforge `engine.run_tiled_parallel` (engine.py:423-505): per query
// block the online row-normalisation protocol carries row scales across key blocks and rescales
// the accumulator (engine.py:481-489); the epilogue divides by the row sum (attention.py:569).
//
// Shape of the kernel (one CTA per SM, 10 warps):
//   warps 0-3  : "row" warpgroup for query tile 0 (rows q0 .. q0+127)
//   warps 4-7  : "row" warpgroup for query tile 1 (rows q0+128 .. q0+255)
//   warp  8    : TMA producer (Q once, then a K/V ring of kStages)
//   warp  9    : TMEM allocator + single-thread tcgen05.mma issuer
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+DV) O1 [256+DV, 256+2DV).
// S_t = Q_t K^T lands in TMEM (fp32), the row warpgroup pulls one score row per thread
// (tcgen05.ld 32x32b), applies the hook epilogue in registers, writes P back into the S columns as
// packed bf16, and the MMA warp consumes P straight from TMEM (A-from-TMEM) for O_t += P V.
// The two query tiles ping-pong so the tensor pipe runs tile 1's MMAs while tile 0's row math runs.
#pragma once
#include <climits>
#include <cuda.h>
#include "params.h"
#include "sm100.cuh"

namespace af {

// Developer timeline trace (-DAF_FWD_TRACE): SM clock stamps of one CTA's row warps / MMA warp,
// read back with af_debug_fwd_trace.  Compiled out of the product build.
#ifdef AF_FWD_TRACE
__device__ unsigned long long g_fwd_trace[9 * 64 * 6 + 1];
#define AF_TRACE(slot, n, ev)                                                              \
  do {                                                                                     \
    if (blockIdx.x == 0 && blockIdx.y == 37 && lane_id() == 0 && (n) < 64)                \
      g_fwd_trace[((slot) * 64 + (n)) * 6 + (ev)] = clock64();                             \
  } while (0)
#else
#define AF_TRACE(slot, n, ev) \
  do {                        \
  } while (0)
#endif
#ifndef AF_FWD_TREEMAX
#define AF_FWD_TREEMAX 1
#endif
#ifndef AF_FWD_EARLY_P
#define AF_FWD_EARLY_P 1
#endif
#ifndef AF_FWD_ALTERNATE
#define AF_FWD_ALTERNATE 1  // softmax rows: the two tiles take turns through the exponentials
#endif
#ifndef AF_SIGMOID_TANH
#define AF_SIGMOID_TANH 1
#endif
#ifndef AF_EXP2_POLY_MASK
#define AF_EXP2_POLY_MASK 14  // column pairs with (c & mask) == 0 use exp2_poly: 14 -> 12.5 %
#endif
constexpr int kBlockM = 128;  // query rows per tile (TMEM lanes)
constexpr int kBlockN = 128;  // keys per block
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

template <int D, int DV, int kStages>
struct FwdSmem {
  static constexpr int kQBytes = kBlockM * D * 2;
  static constexpr int kKBytes = kBlockN * D * 2;
  static constexpr int kVBytes = kBlockN * DV * 2;
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + 2 * kQBytes;
  static constexpr int kVOff = kKOff + kStages * kKBytes;
  static constexpr int kBarOff = kVOff + kStages * kVBytes;
  // barriers: q_full, k_full[S], k_empty[S], v_full[S], v_empty[S], s_full[2], p_full[2], o_done[2]
  static constexpr int kNumBars = 1 + 4 * kStages + 8;  // + p_half[2]
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kRowSumOff = kTmemSlotOff + 16;  // [2 tiles][2 halves][128] fp32
  static constexpr int kRowMaxOff = kRowSumOff + 2 * 2 * 128 * 4;  // [2 bufs][2][2][128] fp32
  static constexpr int kTotal = kRowMaxOff + 2 * 2 * 2 * 128 * 4 + 1024;  // + alignment slack
};

// Each score row is split over two warps (64 key columns each; 16 row warps): twice the warps
// per scheduler to hide the SFU / issue latency of the row epilogue, which otherwise leaves the
// tensor pipe waiting for P.  Softmax exchanges the block row max between the two warps of a row
// once per key block (named barrier per warp pair); row sums are combined once at the end.
#ifndef AF_FWD_SOFTMAX_SPLIT
#define AF_FWD_SOFTMAX_SPLIT 1  // swept: 2 (16 row warps) is no faster for softmax
#endif
__host__ __device__ constexpr int fwd_row_split(int family) {
  return family == kFamilySoftmax ? AF_FWD_SOFTMAX_SPLIT : 2;
}
__host__ __device__ constexpr int fwd_threads(int family) {
  return 32 * (8 * fwd_row_split(family) + 2);
}
AF_DEVICE uint32_t fwd_split_col(int kk) { return kk < 4 ? kk * 8 : 64 + (kk - 4) * 8; }

struct TileBand {
  int jb_lo, jb_hi;  // key-block range [jb_lo, jb_hi)
};

// Range of key blocks any row in [r0, r1) can see under the band mask.
__host__ __device__ inline TileBand key_band(const MaskParams& m, int r0, int r1, int seq_k) {
  int hi = seq_k;
  if (m.causal) hi = min(hi, r1 - 1 + m.diag_offset + 1);
  int lo = 0;
  if (m.window > 0) lo = max(0, r0 + m.diag_offset - m.window + 1);
  TileBand b;
  if (hi <= lo) {
    b.jb_lo = 0;
    b.jb_hi = 0;
  } else {
    b.jb_lo = lo / kBlockN;
    b.jb_hi = (hi + kBlockN - 1) / kBlockN;
  }
  return b;
}

// True when every (i, j) of the block is kept by the band mask and in bounds.
AF_DEVICE bool block_fully_kept(const MaskParams& m, int r0, int c0, int seq_k) {
  if (c0 + kBlockN > seq_k) return false;
  if (m.causal && c0 + kBlockN - 1 > r0 + m.diag_offset) return false;
  if (m.window > 0 && (r0 + kBlockM - 1) + m.diag_offset - c0 >= m.window) return false;
  return true;
}
// True when no (i, j) of the tile's block is kept: a two-tile CTA walks the union of its tiles'
// key bands, so the first / last block of a sliding-window or causal sweep can be empty for one
// tile (its P is zero; the row warps skip the epilogue math).
AF_DEVICE bool block_fully_masked(const MaskParams& m, int r0, int c0, int seq_k) {
  if (c0 >= seq_k) return true;
  if (m.causal && c0 > r0 + kBlockM - 1 + m.diag_offset) return true;
  if (m.window > 0 && c0 + kBlockN - 1 < r0 + m.diag_offset - m.window + 1) return true;
  return false;
}
// Branch-free band test: keep iff lo <= j < hi, with the row's bounds loop-invariant so unrolled
// callers hoist them (short-circuit forms compiled to a branch + reconvergence per score).
AF_DEVICE bool kept(const MaskParams& m, int i, int j, int seq_k) {
  const int hi = m.causal ? min(seq_k, i + m.diag_offset + 1) : seq_k;
  const int lo = m.window > 0 ? i + m.diag_offset - m.window + 1 : INT_MIN;
  return (j >= lo) & (j < hi);
}

template <int kAct>
AF_DEVICE float apply_act(float z) {
  if constexpr (kAct == kActSigmoid) {
#if AF_SIGMOID_TANH
    // sigma(z) = 1/2 + tanh(z / 2) / 2: one MUFU op (tanh.approx, max rel. error ~2^-11, below
    // bf16's 2^-8) and one FFMA — the 1 / (1 + 2^(-z log2 e)) form below spends the MUFU op on
    // ex2 and ~7 FMA-pipe instructions on its reciprocal, and the sigmoid row epilogues are
    // issue-bound (cfg3 K2f: P took 2.2k of a 3.7k-clk iteration).
    return fmaf(0.5f, tanh_approx(0.5f * z), 0.5f);
#else
    // 1 / (1 + 2^(-z log2 e)): one MUFU op (ex2) and the reciprocal on the FMA pipe (rcp_nr) —
    // with rcp.approx as well the sigmoid row epilogue issued two MUFU ops per score, twice the
    // tensor pipe's time per block (16 MUFU lanes / clk / SM); __frcp_rn's IEEE fix-up path is
    // ~10x slower still.  -z log2 e is clamped at 126 so 1 + e stays in rcp_nr's range.
    return rcp_nr(1.0f + ex2(fminf(-z * kLog2e, 126.0f)));
#endif
  } else if constexpr (kAct == kActRelu) {
    return fmaxf(z, 0.0f);
  } else if constexpr (kAct == kActRelu2) {
    const float r = fmaxf(z, 0.0f);
    return r * r;
  } else {
    return z;
  }
}

template <int D, int DV, int kFamily, int kAct, int kStages>
__global__ void __launch_bounds__(fwd_threads(kFamily), 1)
    parallel_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                        const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v,
                        const __grid_constant__ CUtensorMap tm_o, const ParallelFwdParams p) {
  using L = FwdSmem<D, DV, kStages>;
  static_assert(D % 64 == 0 && DV % 64 == 0 && D <= 256 && DV <= 128, "tile dims");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + kStages;
  uint64_t* v_full = k_empty + kStages;
  uint64_t* v_empty = v_full + kStages;
  uint64_t* s_full = v_empty + kStages;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_done = p_full + 2;
  uint64_t* p_half = o_done + 2;  // first 64 keys of P published (one-warp softmax rows)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);
  float* sRowSum = reinterpret_cast<float*>(smem + L::kRowSumOff);
  float* sRowMax = reinterpret_cast<float*>(smem + L::kRowMaxOff);
  constexpr int kSplit = fwd_row_split(kFamily);
  constexpr int kTmaWarp = 8 * kSplit, kMmaWarp = 8 * kSplit + 1;

  const int warp = static_cast<int>(warp_id());
  const int q_blocks = (p.seq_q + 2 * kBlockM - 1) / (2 * kBlockM);
  // Heaviest (latest) query blocks first: causal work grows with the block index.
  const int qb = p.mask.causal ? (q_blocks - 1 - static_cast<int>(blockIdx.x))
                               : static_cast<int>(blockIdx.x);
  const int bh = blockIdx.y;
  const int b = bh / p.heads_q;
  const int h = bh % p.heads_q;
  const int hk = h / (p.heads_q / p.heads_kv);
  const int q0 = qb * 2 * kBlockM;
  const int q_end = min(p.seq_q, q0 + 2 * kBlockM);
  const TileBand band = key_band(p.mask, q0, q_end, p.seq_k);
  const int nk = band.jb_hi - band.jb_lo;

  if (warp == kTmaWarp && lane_id() == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 4 * kSplit);  // one arrival per row warp
      mbar_init(&o_done[t], 1);
      mbar_init(&p_half[t], 4);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kTmaWarp) {
    // ───────────── TMA producer ─────────────
    if (elect_one() && nk > 0) {
      mbar_expect_tx(q_full, 2 * L::kQBytes);
      for (int t = 0; t < 2; ++t)
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(sQ + t * L::kQBytes + c * (kBlockM * 128), &tm_q, q_full, c * 64,
                      q0 + t * kBlockM, h, b);
      for (int n = 0; n < nk; ++n) {
        const int s = n % kStages;
        const uint32_t ph = (n / kStages) & 1;
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
  } else if (warp == kMmaWarp) {
    // ───────────── MMA issuer ─────────────
    if (elect_one() && nk > 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(kBlockM, kBlockN, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(kBlockM, DV, false, true);
      const uint32_t sq_addr = smem_u32(sQ);
      const uint32_t sk_addr = smem_u32(sK);
      const uint32_t sv_addr = smem_u32(sV);
      auto issue_s = [&](int t, int n) {
        const int s = n % kStages;
        const uint32_t d_tmem = tmem + t * kBlockN;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * (kBlockM * 128) + (kk % 4) * 32;
          const uint64_t a = make_sdesc(sq_addr + t * L::kQBytes + off, 0, 1024);
          const uint64_t bdesc = make_sdesc(sk_addr + s * L::kKBytes + (kk / 4) * (kBlockN * 128) +
                                                (kk % 4) * 32,
                                            0, 1024);
          mma_ss(d_tmem, a, bdesc, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[t]);
      };
      // PV over key slices [k_lo, k_hi) of the block (16 keys per MMA)
      auto issue_pv_part = [&](int t, int n, int k_lo, int k_hi) {
        const int s = n % kStages;
        const uint32_t d_tmem = tmem + 2 * kBlockN + t * DV;
        const uint32_t p_tmem = tmem + t * kBlockN;
#pragma unroll
        for (int kk = k_lo; kk < k_hi; ++kk) {
          const uint64_t bdesc =
              make_sdesc(sv_addr + s * L::kVBytes + kk * 16 * 128, kBlockN * 128, 1024);
          mma_ts(d_tmem, p_tmem + (kSplit == 2 ? fwd_split_col(kk) : kk * 8), bdesc, idesc_o,
                 (n > 0 || kk > 0) ? 1u : 0u);
        }
      };
      // One-warp softmax rows publish P in two halves: the first half of PV starts while the
      // row warps are still exponentiating the second half.
      auto wait_p_and_pv = [&](int t, int n) {
        if constexpr (kSplit == 1 && AF_FWD_EARLY_P) {
          mbar_wait(&p_half[t], n & 1);
          tc_fence_after();
          issue_pv_part(t, n, 0, kBlockN / 32);
          mbar_wait(&p_full[t], n & 1);
          tc_fence_after();
          issue_pv_part(t, n, kBlockN / 32, kBlockN / 16);
        } else {
          mbar_wait(&p_full[t], n & 1);
          tc_fence_after();
          issue_pv_part(t, n, 0, kBlockN / 16);
        }
        mma_commit(&o_done[t]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      mma_commit(&k_empty[0]);
      for (int n = 0; n < nk; ++n) {
        const int s = n % kStages;
        const uint32_t ph = (n / kStages) & 1;
        const bool more = n + 1 < nk;
        const int s1 = (n + 1) % kStages;
        const uint32_t ph1 = ((n + 1) / kStages) & 1;
        mbar_wait(&v_full[s], ph);
        AF_TRACE(8, n, 0);
        wait_p_and_pv(0, n);
        AF_TRACE(8, n, 1);
        if (more) {
          mbar_wait(&k_full[s1], ph1);
          tc_fence_after();
          issue_s(0, n + 1);
        }
        wait_p_and_pv(1, n);
        AF_TRACE(8, n, 2);
        mma_commit(&v_empty[s]);
        if (more) {
          issue_s(1, n + 1);
          mma_commit(&k_empty[s1]);
        }
      }
    }
  } else if constexpr (kSplit == 2) {
    // ───────────── row warps, two per score row (non-softmax families) ─────────────
    const int t = warp / 8;          // query tile
    const int wq = warp % 4;         // TMEM lane quarter
    const int ch = (warp / 4) % 2;   // key-column half of the 128-wide block
    const int row = wq * 32 + static_cast<int>(lane_id());
    const int i = q0 + t * kBlockM + row;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t s_tmem = tmem + lane_base + t * kBlockN + ch * 64;
    const uint32_t o_tmem = tmem + lane_base + 2 * kBlockN + t * DV + ch * (DV / 2);
    const int r0 = q0 + t * kBlockM;
    const float slope = (p.slope != nullptr) ? p.slope[h] : 0.0f;
    const float fi = static_cast<float>(i);
    float l_run = 0.0f;
    float m_run = -INFINITY;  // softmax: running max (log2 units), identical in both row halves
    const int pair_bar = 3 + t * 4 + wq;  // named barrier of the two warps sharing these rows
    if constexpr (kFamily == kFamilySoftmax) {
      constexpr bool kCap = kAct == kActSoftcap;
      const float cap_in = p.cap_b * p.scale, cap_out = p.cap_a * kLog2e;
      for (int n = 0; n < nk; ++n) {
        const int c0 = (band.jb_lo + n) * kBlockN;
        const int cb = c0 + ch * 64;
        mbar_wait(&s_full[t], n & 1);
        if (ch == 0) AF_TRACE(t * 4 + wq, n, 0);
        tc_fence_after();
        uint32_t sr[64];
        tmem_ld32(s_tmem, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        tmem_ld32(s_tmem + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_ld_wait();
        if (ch == 0) AF_TRACE(t * 4 + wq, n, 1);
        float* s = reinterpret_cast<float*>(sr);
        const bool full = block_fully_kept(p.mask, r0, c0, p.seq_k);
        const bool fast = !kCap && full && p.scale_log2 > 0.0f;
        float bmax = -INFINITY;
        if (fast) {
#pragma unroll
          for (int c = 0; c < 64; ++c) bmax = fmaxf(bmax, s[c]);
          bmax *= p.scale_log2;
        } else {
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            const float x = kCap ? cap_out * tanh_precise(cap_in * s[c]) : s[c] * p.scale_log2;
            s[c] = (full | kept(p.mask, i, cb + c, p.seq_k)) ? x : -INFINITY;
            bmax = fmaxf(bmax, s[c]);
          }
        }
        // block row max over both halves (double-buffered slot: the partner's next write goes
        // to the other buffer, and the one after that follows its read of this one)
        float* mx = sRowMax + (n & 1) * 512 + t * 256;
        mx[ch * 128 + row] = bmax;
        named_bar_sync(pair_bar, 64);
        bmax = fmaxf(bmax, mx[(1 - ch) * 128 + row]);
        if (ch == 0) AF_TRACE(t * 4 + wq, n, 2);
        const float m_new = fmaxf(m_run, bmax);
        const bool need = (m_new - m_run) > 8.0f;  // lazy rescale, as in the one-warp path
        float factor = 1.0f;
        if (need) {
          factor = (m_run == -INFINITY) ? 0.0f : ex2(m_run - m_new);
          m_run = m_new;
        }
        const float m_use = (m_run == -INFINITY) ? 0.0f : m_run;
        // P in two 32-column chunks, each stored as soon as it is packed (keeps the live
        // register set at the S row plus 16 packed words)
        float lsum;
        if (fast) {
          const float2 sc2 = splat2(p.scale_log2), nm2 = splat2(-m_use);
          float2 ls2[2] = {splat2(0.0f), splat2(0.0f)};
#pragma unroll
          for (int hc = 0; hc < 2; ++hc) {
            uint32_t pk[16];
#pragma unroll
            for (int c = hc * 32; c < hc * 32 + 32; c += 2) {
              const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
              const bool poly = (c & AF_EXP2_POLY_MASK) == 0;
              const float2 e = poly ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
              ls2[(c / 2) & 1] = fadd2(ls2[(c / 2) & 1], e);
              pk[(c / 2) % 16] = pack_bf16(e.x, e.y);
            }
            tmem_st16(s_tmem + hc * 16, pk);
          }
          lsum = (ls2[0].x + ls2[1].x) + (ls2[0].y + ls2[1].y);
        } else {
          lsum = 0.0f;
#pragma unroll
          for (int hc = 0; hc < 2; ++hc) {
            uint32_t pk[16];
#pragma unroll
            for (int c = hc * 32; c < hc * 32 + 32; c += 2) {
              const float e0 = ex2(s[c] - m_use);
              const float e1 = ex2(s[c + 1] - m_use);
              lsum += e0 + e1;
              pk[(c / 2) % 16] = pack_bf16(e0, e1);
            }
            tmem_st16(s_tmem + hc * 16, pk);
          }
        }
        l_run = l_run * factor + lsum;
        tmem_st_wait();
        if (ch == 0) AF_TRACE(t * 4 + wq, n, 3);
        // correction of this warp's O columns (only rows whose max moved by > 2^8)
        if (n > 0 && __any_sync(0xffffffffu, need)) {
          mbar_wait(&o_done[t], (n - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < DV / 64; ++c) {
            uint32_t orr[32];
            tmem_ld32(o_tmem + c * 32, orr);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e)
              orr[e] = __float_as_uint(__uint_as_float(orr[e]) * factor);
            tmem_st32(o_tmem + c * 32, orr);
          }
          tmem_st_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&p_full[t]);
        if (ch == 0) AF_TRACE(t * 4 + wq, n, 5);
      }
    } else
    for (int n = 0; n < nk; ++n) {
      const int c0 = (band.jb_lo + n) * kBlockN;
      const int cb = c0 + ch * 64;
      mbar_wait(&s_full[t], n & 1);
      tc_fence_after();
      if (block_fully_masked(p.mask, r0, c0, p.seq_k)) {  // P = 0 without the epilogue math
        uint32_t z[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) z[e] = 0u;
        tmem_st32(s_tmem, z);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&p_full[t]);
        continue;
      }
      uint32_t sr[64];
      tmem_ld32(s_tmem, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      tmem_ld32(s_tmem + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
      tmem_ld_wait();
      const float* s = reinterpret_cast<const float*>(sr);
      const bool full = block_fully_kept(p.mask, r0, c0, p.seq_k);
      uint32_t pk[32];
      if constexpr (kFamily == kFamilyAbssum) {
        const float base = (fi - static_cast<float>(cb)) * slope;
        float asum = 0.0f;
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          float e0 = s[c] * p.scale * ex2(base - slope * static_cast<float>(c));
          float e1 = s[c + 1] * p.scale * ex2(base - slope * static_cast<float>(c + 1));
          if (!full) {
            if (!kept(p.mask, i, cb + c, p.seq_k)) e0 = 0.0f;
            if (!kept(p.mask, i, cb + c + 1, p.seq_k)) e1 = 0.0f;
          }
          asum += fabsf(e0) + fabsf(e1);
          pk[c / 2] = pack_bf16(e0, e1);
        }
        l_run += asum;
      } else {
        const float bias = p.bias + slope * static_cast<float>(cb) - slope * fi;
        if (full) {  // compact fast path: no per-element mask tests
#pragma unroll
          for (int c = 0; c < 64; c += 2)
            pk[c / 2] =
                pack_bf16(apply_act<kAct>(s[c] * p.scale + bias + slope * static_cast<float>(c)),
                          apply_act<kAct>(s[c + 1] * p.scale + bias +
                                          slope * static_cast<float>(c + 1)));
        } else {
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            float e0 = apply_act<kAct>(s[c] * p.scale + bias + slope * static_cast<float>(c));
            float e1 =
                apply_act<kAct>(s[c + 1] * p.scale + bias + slope * static_cast<float>(c + 1));
            if (!kept(p.mask, i, cb + c, p.seq_k)) e0 = 0.0f;
            if (!kept(p.mask, i, cb + c + 1, p.seq_k)) e1 = 0.0f;
            pk[c / 2] = pack_bf16(e0, e1);
          }
        }
      }
      // packed P of this key half over its own S columns (the PV MMA reads fwd_split_col)
      tmem_st32(s_tmem, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&p_full[t]);
    }
    // ───────────── epilogue: O (this warp's DV/2 columns), abssum row statistic ─────────────
    float inv = 1.0f;
    if constexpr (kFamily == kFamilySoftmax) {
      sRowSum[(t * 2 + ch) * 128 + row] = l_run;
      named_bar_sync(pair_bar, 64);
      const float total = sRowSum[t * 2 * 128 + row] + sRowSum[(t * 2 + 1) * 128 + row];
      inv = (total == 0.0f) ? 0.0f : 1.0f / total;
      if (ch == 0 && p.lse != nullptr && i < p.seq_q)
        p.lse[(static_cast<int64_t>(b) * p.heads_q + h) * p.seq_q + i] =
            (total == 0.0f) ? -INFINITY : (m_run * kLn2 + logf(total));
    }
    if constexpr (kFamily == kFamilyAbssum) {
      sRowSum[(t * 2 + ch) * 128 + row] = l_run;
      named_bar_sync(1 + t, 256);
      const float total = sRowSum[t * 2 * 128 + row] + sRowSum[(t * 2 + 1) * 128 + row];
      if (p.cap_a != 0.0f) inv = 1.0f / fmaxf(total, 1.0f);
      if (ch == 0 && p.lse != nullptr && i < p.seq_q)
        p.lse[(static_cast<int64_t>(b) * p.heads_q + h) * p.seq_q + i] = total;
    }
    if (nk > 0) {
      mbar_wait(&o_done[t], (nk - 1) & 1);
      tc_fence_after();
    }
    __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o) + b * p.o_stride_b +
                          h * p.o_stride_h + static_cast<int64_t>(i) * p.o_stride_s +
                          ch * (DV / 2);
    // O through the tile's Q buffer (free: every S MMA of this tile has completed) as SW128
    // [rows][64] boxes and TMA stores — per-thread 16-byte stores to 32 different rows per
    // instruction cost LSU / L2 sector work at the end of every CTA
    constexpr bool kStageO = DV / 2 == 64;
    const bool stage_o = kStageO && p.o_tma != 0;
    uint8_t* sO = sQ + t * L::kQBytes;
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
      if (stage_o) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int g = c * 4 + v;  // 16-byte chunk of the 64-column box (box = ch)
          *reinterpret_cast<uint4*>(sO + ch * (kBlockM * 128) + row * 128 +
                                    ((g ^ (row & 7)) << 4)) = make_uint4(
              pack_bf16(__uint_as_float(orr[v * 8 + 0]) * inv, __uint_as_float(orr[v * 8 + 1]) * inv),
              pack_bf16(__uint_as_float(orr[v * 8 + 2]) * inv, __uint_as_float(orr[v * 8 + 3]) * inv),
              pack_bf16(__uint_as_float(orr[v * 8 + 4]) * inv, __uint_as_float(orr[v * 8 + 5]) * inv),
              pack_bf16(__uint_as_float(orr[v * 8 + 6]) * inv, __uint_as_float(orr[v * 8 + 7]) * inv));
        }
      } else if (i < p.seq_q) {
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
    if (stage_o) {  // this warp's 32 rows of box ch (rows past seq_q are clipped by the map)
      fence_proxy_async_smem();
      __syncwarp();
      if (lane_id() == 0) {
        tma_store_4d(&tm_o, sO + ch * (kBlockM * 128) + wq * 32 * 128, ch * 64,
                     r0 + wq * 32, h, b);
        bulk_commit();
        bulk_wait<0>();
      }
    }
  } else {
    // ───────────── row warpgroups (hook epilogue) ─────────────
    const int t = warp / 4;                  // query tile
    const int wq = warp % 4;                 // TMEM lane quarter
    const int row = wq * 32 + static_cast<int>(lane_id());
    const int i = q0 + t * kBlockM + row;    // absolute query index
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t s_tmem = tmem + lane_base + t * kBlockN;
    const uint32_t o_tmem = tmem + lane_base + 2 * kBlockN + t * DV;
    const int r0 = q0 + t * kBlockM;

    float m_run = -INFINITY;  // running max, log2-scaled units
    float l_run = 0.0f;
    float slope = 0.0f;
    if constexpr (kFamily != kFamilySoftmax) {
      if (p.slope != nullptr) slope = p.slope[h];
    }
    const float fi = static_cast<float>(i);

    for (int n = 0; n < nk; ++n) {
      const int c0 = (band.jb_lo + n) * kBlockN;
      mbar_wait(&s_full[t], n & 1);
      AF_TRACE(t * 4 + wq, n, 0);
      tc_fence_after();
      uint32_t sr[kBlockN];
#pragma unroll
      for (int c = 0; c < kBlockN / 32; ++c)
        tmem_ld32(s_tmem + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_ld_wait();
      AF_TRACE(t * 4 + wq, n, 1);
      float* s = reinterpret_cast<float*>(sr);
      const bool full = block_fully_kept(p.mask, r0, c0, p.seq_k);

      if constexpr (kFamily == kFamilySoftmax) {
        // Fully-kept blocks (the bulk of a causal sweep): the row max is taken on the raw scores
        // and the scale folds into one FFMA per element; an eighth of the exponentials run as a
        // polynomial on the FMA pipe so the MUFU stream stays below the MMA time.
        constexpr bool kCap = kAct == kActSoftcap;
        const bool fast = !kCap && full && p.scale_log2 > 0.0f;
        const float cap_in = p.cap_b * p.scale, cap_out = p.cap_a * kLog2e;
        float bmax = -INFINITY;
        if (fast) {
#if AF_FWD_TREEMAX
          // four independent FMNMX3 chains (a single chain is 64 dependent max ops)
          float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < kBlockN; c += 2)
            mx4[(c / 2) & 3] = fmaxf(mx4[(c / 2) & 3], fmaxf(s[c], s[c + 1]));
          bmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
#else
#pragma unroll
          for (int c = 0; c < kBlockN; ++c) bmax = fmaxf(bmax, s[c]);
#endif
          bmax *= p.scale_log2;
        } else {
#pragma unroll
          for (int c = 0; c < kBlockN; ++c) {
            const float x = kCap ? cap_out * tanh_precise(cap_in * s[c]) : s[c] * p.scale_log2;
            s[c] = (full | kept(p.mask, i, c0 + c, p.seq_k)) ? x : -INFINITY;
            bmax = fmaxf(bmax, s[c]);
          }
        }
        const float m_new = fmaxf(m_run, bmax);
        // Lazy rescale: keep the stale max unless the new one exceeds it by more than 2^8.
        const bool need = (m_new - m_run) > 8.0f;
        float factor = 1.0f;
        if (need) {
          factor = (m_run == -INFINITY) ? 0.0f : ex2(m_run - m_new);
          m_run = m_new;
        }
        const float m_use = (m_run == -INFINITY) ? 0.0f : m_run;
        AF_TRACE(t * 4 + wq, n, 2);
        // P in two 64-key halves; the first is published (p_half) before the second is
        // exponentiated, so the MMA warp runs half of PV under the row warps' second half.
        // The O correction (only rows whose max moved by > 2^8) precedes the first publish: PV(n)
        // must accumulate onto the rescaled O, and PV(n-1) has completed (S(n) was issued behind
        // it); it runs after half of the S row is dead, to keep the register peak down.
        auto publish = [&](int hh, const uint32_t (&pk)[kBlockN / 4]) {
          tmem_st32(s_tmem + hh * 32, pk);
          tmem_st_wait();
          if (hh == 0 && n > 0 && __any_sync(0xffffffffu, need)) {
            mbar_wait(&o_done[t], (n - 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < DV / 32; ++c) {
              uint32_t orr[32];
              tmem_ld32(o_tmem + c * 32, orr);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e)
                orr[e] = __float_as_uint(__uint_as_float(orr[e]) * factor);
              tmem_st32(o_tmem + c * 32, orr);
            }
            tmem_st_wait();
          }
          if (hh == 0 && AF_FWD_EARLY_P) {
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&p_half[t]);
            AF_TRACE(t * 4 + wq, n, 3);
          }
        };
        // The two query tiles' row warps of a lane quarter share a scheduler and its MUFU lanes:
        // they take turns through the exponential phase (tile 0 block n, tile 1 block n, tile 0
        // block n+1, ...; a named-barrier token per direction) instead of contending in it —
        // traced: both phases overlapping ran each at half the MUFU rate (≈2.1k clk softmax per
        // tile, 3.4k clk period).
        if constexpr (AF_FWD_ALTERNATE) {
          if (t == 0) {
            if (n > 0) named_bar_sync(5 + wq, 64);  // tile 1 is through block n-1
          } else {
            named_bar_sync(1 + wq, 64);  // tile 0 is through block n
          }
        }
        float2 ls2[2] = {splat2(0.0f), splat2(0.0f)};
        if (fast) {
          // packed pairs: one FFMA2 for the scale/max fold, FADD2 row sums (two chains); an
          // eighth of the exponentials on the FMA pipe (exp2_poly2)
          const float2 sc2 = splat2(p.scale_log2), nm2 = splat2(-m_use);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t pk[kBlockN / 4];
#pragma unroll
            for (int c = hh * (kBlockN / 2); c < (hh + 1) * (kBlockN / 2); c += 2) {
              const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
              const bool poly = (c & AF_EXP2_POLY_MASK) == 0;  // default: c % 16 in {0, 1}
              const float2 e = poly ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
              ls2[(c / 2) & 1] = fadd2(ls2[(c / 2) & 1], e);
              pk[(c / 2) % (kBlockN / 4)] = pack_bf16(e.x, e.y);
            }
            publish(hh, pk);
          }
        } else {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t pk[kBlockN / 4];
#pragma unroll
            for (int c = hh * (kBlockN / 2); c < (hh + 1) * (kBlockN / 2); c += 2) {
              const float2 e = make_float2(ex2(s[c] - m_use), ex2(s[c + 1] - m_use));
              ls2[(c / 2) & 1] = fadd2(ls2[(c / 2) & 1], e);
              pk[(c / 2) % (kBlockN / 4)] = pack_bf16(e.x, e.y);
            }
            publish(hh, pk);
          }
        }
        l_run = l_run * factor + ((ls2[0].x + ls2[1].x) + (ls2[0].y + ls2[1].y));
        if constexpr (AF_FWD_ALTERNATE) named_bar_arrive(t == 0 ? 1 + wq : 5 + wq, 64);
        AF_TRACE(t * 4 + wq, n, 4);
      } else if constexpr (kFamily == kFamilyAbssum) {
        // s = tau q.k gamma^(i-j) on the kept band (slope = log2 gamma); l_run = sum |s|
        uint32_t pk[kBlockN / 2];
        const float base = (fi - static_cast<float>(c0)) * slope;
        float asum = 0.0f;
#pragma unroll
        for (int c = 0; c < kBlockN; c += 2) {
          float e0 = s[c] * p.scale * ex2(base - slope * static_cast<float>(c));
          float e1 = s[c + 1] * p.scale * ex2(base - slope * static_cast<float>(c + 1));
          if (!full) {
            if (!kept(p.mask, i, c0 + c, p.seq_k)) e0 = 0.0f;
            if (!kept(p.mask, i, c0 + c + 1, p.seq_k)) e1 = 0.0f;
          }
          asum += fabsf(e0) + fabsf(e1);
          pk[c / 2] = pack_bf16(e0, e1);
        }
        l_run += asum;
#pragma unroll
        for (int c = 0; c < kBlockN / 64; ++c)
          tmem_st32(s_tmem + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[c * 32]));
        tmem_st_wait();
      } else {
        uint32_t pk[kBlockN / 2];
        const float bias = p.bias + slope * static_cast<float>(c0) - slope * fi;
#pragma unroll
        for (int c = 0; c < kBlockN; c += 2) {
          float z0 = s[c] * p.scale + bias + slope * static_cast<float>(c);
          float z1 = s[c + 1] * p.scale + bias + slope * static_cast<float>(c + 1);
          float e0 = apply_act<kAct>(z0);
          float e1 = apply_act<kAct>(z1);
          if (!full) {
            if (!kept(p.mask, i, c0 + c, p.seq_k)) e0 = 0.0f;
            if (!kept(p.mask, i, c0 + c + 1, p.seq_k)) e1 = 0.0f;
          }
          pk[c / 2] = pack_bf16(e0, e1);
        }
#pragma unroll
        for (int c = 0; c < kBlockN / 64; ++c)
          tmem_st32(s_tmem + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[c * 32]));
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&p_full[t]);
      AF_TRACE(t * 4 + wq, n, 5);
    }

    // ───────────── epilogue: O / l, LSE ─────────────
    if constexpr (kFamily == kFamilySoftmax && AF_FWD_ALTERNATE) {
      if (t == 0 && nk > 0) named_bar_sync(5 + wq, 64);  // tile 1's last token
    }
    float inv = 1.0f;
    if constexpr (kFamily == kFamilySoftmax) inv = (l_run == 0.0f) ? 0.0f : 1.0f / l_run;
    if constexpr (kFamily == kFamilyAbssum) {
      if (p.cap_a != 0.0f) inv = 1.0f / fmaxf(l_run, 1.0f);
    }
    if (nk > 0) {
      mbar_wait(&o_done[t], (nk - 1) & 1);
      tc_fence_after();
    }
    __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o) + b * p.o_stride_b +
                          h * p.o_stride_h + static_cast<int64_t>(i) * p.o_stride_s;
    // O through the tile's Q buffer (see the two-warp path above) when the map exists
    const bool stage_o = p.o_tma != 0;
    uint8_t* sO = sQ + t * L::kQBytes;
#pragma unroll
    for (int c = 0; c < DV / 32; ++c) {
      uint32_t orr[32];
      if (nk > 0) {
        tmem_ld32(o_tmem + c * 32, orr);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) orr[e] = 0u;
      }
      if (stage_o) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int g = (c % 2) * 4 + v;  // 16-byte chunk of 64-column box c / 2
          *reinterpret_cast<uint4*>(sO + (c / 2) * (kBlockM * 128) + row * 128 +
                                    ((g ^ (row & 7)) << 4)) = make_uint4(
              pack_bf16(__uint_as_float(orr[v * 8 + 0]) * inv, __uint_as_float(orr[v * 8 + 1]) * inv),
              pack_bf16(__uint_as_float(orr[v * 8 + 2]) * inv, __uint_as_float(orr[v * 8 + 3]) * inv),
              pack_bf16(__uint_as_float(orr[v * 8 + 4]) * inv, __uint_as_float(orr[v * 8 + 5]) * inv),
              pack_bf16(__uint_as_float(orr[v * 8 + 6]) * inv, __uint_as_float(orr[v * 8 + 7]) * inv));
        }
        continue;
      }
      if (i < p.seq_q) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(orr[v * 8 + 0]) * inv, __uint_as_float(orr[v * 8 + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(orr[v * 8 + 2]) * inv, __uint_as_float(orr[v * 8 + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(orr[v * 8 + 4]) * inv, __uint_as_float(orr[v * 8 + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(orr[v * 8 + 6]) * inv, __uint_as_float(orr[v * 8 + 7]) * inv);
          dst[v] = w;
        }
      }
    }
    if (stage_o) {  // this warp's 32 rows of every 64-column box (rows past seq_q are clipped)
      fence_proxy_async_smem();
      __syncwarp();
      if (lane_id() == 0) {
#pragma unroll
        for (int x = 0; x < DV / 64; ++x)
          tma_store_4d(&tm_o, sO + x * (kBlockM * 128) + wq * 32 * 128, x * 64, r0 + wq * 32, h, b);
        bulk_commit();
        bulk_wait<0>();
      }
    }
    if constexpr (kFamily == kFamilySoftmax) {
      if (p.lse != nullptr && i < p.seq_q) {
        const float lse = (l_run == 0.0f) ? -INFINITY : (m_run * kLn2 + logf(l_run));
        p.lse[(static_cast<int64_t>(b) * p.heads_q + h) * p.seq_q + i] = lse;
      }
    }
    if constexpr (kFamily == kFamilyAbssum) {  // row statistic for the backward: sum_j |s_ij|
      if (p.lse != nullptr && i < p.seq_q)
        p.lse[(static_cast<int64_t>(b) * p.heads_q + h) * p.seq_q + i] = l_run;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace af
