// K3 — MLA attention (DeepSeek-V2: Dqk = 576, Dv = 512, one latent KV head, V = K[:, :512]).
//
// Softmax attention over a shared latent cache, i.e. attnforge `engine.run_tiled_parallel`
// (engine.py:423-505) with the builtin softmax rownorm (attention.py:556-572) on a variant whose
// K/V are one latent head (V aliases the first d_v columns of K).  Two modes:
//   prefill : rows = 128 query positions of one head, causal (top-left), grid over
//             (query tile, head, value half)
//   decode  : rows = the 128 heads of one query token (seq_q = 1, unmasked — SURVEY §0), grid
//             over (batch, key split, value half); splits are merged by mla_combine_kernel.
// Budget: the fp32 O accumulator of 128 rows x 512 would fill all of TMEM, so each CTA owns one
// 256-wide value half (the two halves recompute S; 1.53x the QK^T work).  Both prefill and decode
// stream 32-key latent tiles (36 KB, 4-stage ring): the S double buffer then takes TMEM [0,64)
// only, so Q (128 x 576 bf16) columns [0, 384) sit in TMEM as the A operand of TS MMAs
// ([384,512) and [64,128); no shared-memory A re-reads — at N = 32 the S GEMM is otherwise bound
// by re-reading Q from smem every tile) and only Q[:, 384:576] (48 KB) stays in smem.
// TMEM: S double buffer [0,64) (P packed in place) | Q[:, 256:384] [64,128) | O half [128,384) |
// Q[:, 0:256] [384,512).  (64-key prefill tiles — AF_MLA_PREFILL_N=64 — keep Q[:, 0:256] in TMEM
// and a 2-stage ring; measured 9 + 10 % slower once the softmax rows stopped branching.)
// Warps: 0-3 softmax rows (one row per thread, FA4-style lazy rescale), 4 TMA, 5 MMA.
#pragma once
#include <climits>
#include <cuda.h>
#include "params.h"
#include "sm100.cuh"
#include "parallel_fwd.cuh"

namespace af {

// Developer timeline (-DAF_MLA_TRACE): SM-clock stamps of CTA 0 (the heaviest causal prefill
// tile, value half 0) per key tile, read back with af_debug_mla_trace.
#ifdef AF_MLA_TRACE
#ifndef AF_MLA_TRACE_DECODE
#define AF_MLA_TRACE_DECODE 0  // 1: trace the decode kernel (batch 0, split 0, value half 0)
#endif
__device__ long long g_mla_trace[10][128];
#define MLA_TRACE(ev, n)                                                              \
  do {                                                                                \
    if (kDecode == AF_MLA_TRACE_DECODE && blockIdx.x == 0 && lane_id() == 0 && (n) < 128) \
      g_mla_trace[ev][n] = clock64();                                                 \
  } while (0)
#else
#define MLA_TRACE(ev, n) \
  do {                   \
  } while (0)
#endif

constexpr int kMlaDqk = 576;
constexpr int kMlaDv = 512;
constexpr int kMlaHalf = 256;
// keys per latent tile and ring depth: prefill (KV reused from L2 across heads, compute bound)
// 64-key tiles x 2 stages; decode (KV streamed once from HBM) 32-key tiles x 4 stages, i.e. three
// tiles of prefetch distance, to hide the HBM latency behind the S / softmax / PV chain.
#ifndef AF_MLA_DECODE_QT
#define AF_MLA_DECODE_QT 384
#endif
#ifndef AF_MLA_PREFILL_QT
#define AF_MLA_PREFILL_QT 384  // 32-key prefill tiles leave TMEM [64,128) free for Q[:, 256:384]
#endif
#ifndef AF_MLA_PREFILL_N
#define AF_MLA_PREFILL_N 32  // swept after the branch-free softmax: 32 beats 64 by ~9 %
#endif
#ifndef AF_MLA_DECODE_N
#define AF_MLA_DECODE_N 32
#endif
template <bool kDecode>
struct MlaTile {
  static constexpr int kN = kDecode ? AF_MLA_DECODE_N : AF_MLA_PREFILL_N;
  static constexpr int kStages = kN == 32 ? 4 : 2;
  // Q columns [0, kQT) held in TMEM as TS-MMA A operand; a 32-key S double buffer leaves TMEM
  // columns [64, 128) free for Q columns [256, 384), so fewer S MMAs stream Q from smem
  static constexpr int kQT = kN == 32 ? (kDecode ? AF_MLA_DECODE_QT : AF_MLA_PREFILL_QT) : 256;
};
constexpr int kMlaN = 64;     // prefill tile (split lengths of decode are multiples of both)

struct MlaParams {
  int batch, heads, seq_q, seq_k;
  float scale_log2;
  int causal;
  int splits;            // decode: key splits per batch
  int split_len;         // decode: keys per split (multiple of kMlaN)
  // Q rows for the TMEM part (bf16, element strides [b, h, s]; decode: s = head, h unused)
  const __nv_bfloat16* q;
  int64_t q_sb, q_sh, q_ss;
  // prefill output (bf16 [B, H, Sq, 512], element strides) + LSE [B, H, Sq]
  void* o;
  int64_t o_sb, o_sh, o_ss;
  float* lse;
  int o_tma;  // O (prefill) / partial O (decode) leaves through tm_o (TMA stores of staged boxes)
  // decode partials: fp32 [B, splits, H, 512] and lse [B, splits, H]
  float* part_o;
  float* part_lse;
};

// Shared memory: Q columns [256, 576) as 5 boxes [128 rows][64] (80 KB) + a 2-stage ring of
// 64-key latent tiles (9 boxes [64 keys][64] = 72 KB each).  TMEM (512 columns): S double buffer
// [0, 128) (P packed in place) | O half [128, 384) | Q columns [0, 256) packed bf16 [384, 512).
template <int kN, int kSt, int kQT>
struct MlaSmem {
  static constexpr int kQBox = 128 * 128;
  static constexpr int kKBox = kN * 128;
  static constexpr int kQBytes = (576 - kQT) / 64 * kQBox;
  static constexpr int kKBytes = 9 * kKBox;
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQBytes;
  static constexpr int kBarOff = kKOff + kSt * kKBytes;
  // q_full, q_ready, k_full[kSt], k_empty[kSt], s_full[2], p_ready[2], o_done[2]
  static constexpr int kNumBars = 8 + 2 * kSt;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
};

template <bool kDecode>
__global__ void __launch_bounds__(192, 1)
    mla_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                   const __grid_constant__ CUtensorMap tm_kv,
                   const __grid_constant__ CUtensorMap tm_o,  // prefill O / decode partial O
                   const MlaParams p) {
  constexpr int kN = MlaTile<kDecode>::kN;
  constexpr int kSt = MlaTile<kDecode>::kStages;
  constexpr int kQT = MlaTile<kDecode>::kQT;
  constexpr int kQB = (kMlaDqk - kQT) / 64;  // Q boxes of 64 columns in smem
  static_assert(kQT == 256 || (kQT == 384 && 2 * kN <= 64), "TMEM map");
  using L = MlaSmem<kN, kSt, kQT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sK = smem + L::kKOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* q_ready = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = bars + 2 + kSt;
  uint64_t* s_full = bars + 2 + 2 * kSt;
  // p_ready[n % 2]: a softmax warp may start tile n+1 (S(n+1) is issued before PV(n)) before
  // the slowest warp has published P(n); one barrier would count its arrival toward tile n
  uint64_t* p_ready = s_full + 2;
  // o_done[n % 2]: PV(n) done; exact parity waits need PV(n - 2) done, which S(n + 1) implies
  uint64_t* o_done = p_ready + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);

  const int warp = static_cast<int>(warp_id());
  const int half = blockIdx.x & 1;  // value half: columns [256*half, 256*half + 256)
  int b, h = 0, q0 = 0, split = 0, kv_lo, kv_hi;
  if constexpr (kDecode) {
    const int rest = blockIdx.x >> 1;
    split = rest % p.splits;
    b = rest / p.splits;
    kv_lo = split * p.split_len;
    kv_hi = min(p.seq_k, kv_lo + p.split_len);
  } else {
    const int q_tiles = (p.seq_q + 127) / 128;
    const int rest = blockIdx.x >> 1;
    const int qt_raw = rest % q_tiles;
    const int bh = rest / q_tiles;
    b = bh / p.heads;
    h = bh % p.heads;
    const int qt = p.causal ? q_tiles - 1 - qt_raw : qt_raw;
    q0 = qt * 128;
    kv_lo = 0;
    kv_hi = p.seq_k;
    if (p.causal) kv_hi = min(kv_hi, q0 + 128);
  }
  const int nk = kv_hi > kv_lo ? (kv_hi - kv_lo + kN - 1) / kN : 0;

  if (warp == 4 && lane_id() == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_ready, 4);
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(&p_ready[0], 4);
    mbar_init(&p_ready[1], 4);
    mbar_init(&o_done[0], 1);
    mbar_init(&o_done[1], 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kColO = 128, kColQ = 384;
  // TMEM column of the packed Q chunk c (64 Q columns = 32 packed TMEM columns)
  auto q_tcol = [](int c) -> uint32_t { return c < 4 ? kColQ + c * 32 : 64 + (c - 4) * 32; };

  // Q columns [0, kQT) (bound for TMEM) are staged by TMA at the tail of the latent ring: the row
  // warps copy them into TMEM before the ring reaches those stages (per-thread row loads of
  // 768 bytes each were uncoalesced global reads at the start of every CTA)
  constexpr int kStgOff = kSt * L::kKBytes - (kQT / 64) * L::kQBox;
  static_assert(kStgOff >= 0, "Q staging fits the latent ring");
  if (warp == 4) {
    if (elect_one() && nk > 0) {
      mbar_expect_tx(q_full, L::kQBytes + (kQT / 64) * L::kQBox);
      for (int c = 0; c < kQB + kQT / 64; ++c) {
        const int col = c < kQB ? kQT + c * 64 : (c - kQB) * 64;
        uint8_t* dst = c < kQB ? sQ + c * L::kQBox : sK + kStgOff + (c - kQB) * L::kQBox;
        if constexpr (kDecode)
          tma_load_4d(dst, &tm_q, q_full, col, 0, b, 0);
        else
          tma_load_4d(dst, &tm_q, q_full, col, q0, h, b);
      }
      bool staged = true;
      for (int n = 0; n < nk; ++n) {
        const int s = n % kSt;
        if (staged && (s + 1) * L::kKBytes > kStgOff) {
          mbar_wait(q_ready, 0);  // the staged Q columns are in TMEM
          staged = false;
        }
        mbar_wait(&k_empty[s], ((n / kSt) & 1) ^ 1);
        MLA_TRACE(0, n);
        mbar_expect_tx(&k_full[s], L::kKBytes);
        const int j0 = kv_lo + n * kN;
        for (int c = 0; c < 9; ++c)
          tma_load_4d_hint(sK + s * L::kKBytes + c * L::kKBox, &tm_kv, &k_full[s], c * 64, j0, b,
                           0, kEvictLast);
      }
    }
  } else if (warp == 5) {
    if (elect_one() && nk > 0) {
      constexpr uint32_t id_s = make_idesc_bf16(128, kN, false, false);        // S = Q K^T
      constexpr uint32_t id_o = make_idesc_bf16(128, kMlaHalf, false, true);   // O += P V
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK);
      auto issue_s = [&](int n) {
        const int s = n & 1;  // TMEM S buffer
        const int st = n % kSt;
        mbar_wait(&k_full[st], (n / kSt) & 1);
        MLA_TRACE(1, n);
        tc_fence_after();
        const uint32_t kb = aK + st * L::kKBytes;
#pragma unroll
        for (int kk = 0; kk < kQT / 16; ++kk)  // Q columns [0, kQT) from TMEM
          mma_ts(tmem + s * kN, tmem + q_tcol(kk / 4) + (kk % 4) * 8,
                 make_sdesc(kb + (kk / 4) * L::kKBox + (kk % 4) * 32, 0, 1024), id_s, kk > 0);
#pragma unroll
        for (int kk = kQT / 16; kk < kMlaDqk / 16; ++kk)  // columns [kQT, 576) from smem
          mma_ss(tmem + s * kN,
                 make_sdesc(aQ + (kk / 4 - kQT / 64) * L::kQBox + (kk % 4) * 32, 0, 1024),
                 make_sdesc(kb + (kk / 4) * L::kKBox + (kk % 4) * 32, 0, 1024), id_s, 1u);
        mma_commit(&s_full[s]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(q_ready, 0);
      tc_fence_after();
      issue_s(0);
      for (int n = 0; n < nk; ++n) {
        const int s = n & 1;
        const int st = n % kSt;
        if (n + 1 < nk) issue_s(n + 1);
        mbar_wait(&p_ready[n & 1], (n >> 1) & 1);
        MLA_TRACE(2, n);
        tc_fence_after();
        // V = latent columns [256*half, +256): boxes 4*half .. 4*half+3 of the tile, MN-major
        const uint32_t vbase = aK + st * L::kKBytes + half * 4 * L::kKBox;
#pragma unroll
        for (int kk = 0; kk < kN / 16; ++kk)
          mma_ts(tmem + kColO, tmem + s * kN + kk * 8,
                 make_sdesc(vbase + kk * 2048, L::kKBox, 1024), id_o, (n > 0 || kk > 0));
        mma_commit(&o_done[n & 1]);
        mma_commit(&k_empty[st]);
      }
    }
  } else {
    // ───────────── softmax rows ─────────────
    const int row = warp * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    const int i = kDecode ? 0 : q0 + row;  // query position (prefill)
    {  // Q columns [0, kQT) of this row -> TMEM (packed bf16 pairs, A-operand layout), from the
       // staged SW128 boxes (rows past the tensor were zero-filled by TMA)
      if (nk > 0) mbar_wait(q_full, 0);
#pragma unroll
      for (int c = 0; c < kQT / 64; ++c) {
        uint32_t w[32];
        const uint8_t* bx = sK + kStgOff + c * L::kQBox;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint4 x = *reinterpret_cast<const uint4*>(bx + row * 128 + ((v ^ (row & 7)) << 4));
          w[v * 4 + 0] = x.x;
          w[v * 4 + 1] = x.y;
          w[v * 4 + 2] = x.z;
          w[v * 4 + 3] = x.w;
        }
        tmem_st32(tmem + lane_base + q_tcol(c), w);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(q_ready);
    }
    float m_run = -INFINITY, l_run = 0.0f;
    for (int n = 0; n < nk; ++n) {
      const int s = n & 1;
      const int j0 = kv_lo + n * kN;
      mbar_wait(&s_full[s], (n >> 1) & 1);
      MLA_TRACE(3, n);
      tc_fence_after();
      uint32_t sr[kN];
#pragma unroll
      for (int c = 0; c < kN / 32; ++c)
        tmem_ld32(tmem + lane_base + s * kN + c * 32,
                  *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_ld_wait();
      MLA_TRACE(5, n);
      float x[kN];
      const bool full = (j0 + kN <= kv_hi) && (kDecode || !p.causal || j0 + kN - 1 <= q0);
      // branch-free per element (a short-circuit keep test compiled to a branch + reconvergence
      // per score and made this loop the prefill's critical path: ~3.7k clk per 64-key tile)
      const int lim = full ? INT_MAX : min(kv_hi - j0, (kDecode || !p.causal) ? INT_MAX : i - j0 + 1);
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int e = 0; e < kN; ++e) {
        x[e] = (e < lim) ? __uint_as_float(sr[e]) * p.scale_log2 : -INFINITY;
        mx4[e & 3] = fmaxf(mx4[e & 3], x[e]);
      }
      const float bmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      const float m_new = fmaxf(m_run, bmax);
      const bool need = (m_new - m_run) > 8.0f;
      float factor = 1.0f;
      if (need) {
        factor = (m_run == -INFINITY) ? 0.0f : ex2(m_run - m_new);
        m_run = m_new;
      }
      const float m_use = (m_run == -INFINITY) ? 0.0f : m_run;
      MLA_TRACE(6, n);
      uint32_t pk[kN / 2];
      float lsum = 0.0f;
#pragma unroll
      for (int e = 0; e < kN; e += 2) {
        const float e0 = ex2(x[e] - m_use), e1 = ex2(x[e + 1] - m_use);
        lsum += e0 + e1;
        pk[e / 2] = pack_bf16(e0, e1);
      }
      l_run = l_run * factor + lsum;
      MLA_TRACE(7, n);
      if constexpr (kN == 64)
        tmem_st32(tmem + lane_base + s * kN, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
      else
        tmem_st16(tmem + lane_base + s * kN, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
      tmem_st_wait();
      MLA_TRACE(8, n);
      if (n > 0 && __any_sync(0xffffffffu, need)) {
        mbar_wait(&o_done[(n - 1) & 1], ((n - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < kMlaHalf / 32; ++c) {
          uint32_t orr[32];
          tmem_ld32(tmem + lane_base + kColO + c * 32, orr);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) orr[e] = __float_as_uint(__uint_as_float(orr[e]) * factor);
          tmem_st32(tmem + lane_base + kColO + c * 32, orr);
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&p_ready[n & 1]);
      MLA_TRACE(4, n);
    }
    // ───────────── epilogue ─────────────
    if (nk > 0) {
      mbar_wait(&o_done[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
      tc_fence_after();
    }
    const float inv = (l_run == 0.0f) ? 0.0f : 1.0f / l_run;
    const float lse = (l_run == 0.0f) ? -INFINITY : (m_run * kLn2 + logf(l_run));
    if constexpr (kDecode) {
      // rows are heads; partial (normalised) output of this split
      const int hh = row;
      float* dst = p.part_o + ((static_cast<int64_t>(b) * p.splits + split) * p.heads + hh) * kMlaDv +
                   half * kMlaHalf;
      // fp32 partial rows through the drained latent ring as SW128 [32 rows][32 cols] boxes and
      // TMA stores (eight per warp)
      const bool stage_o = p.o_tma != 0;
      static_assert(kSt * L::kKBytes >= 4 * 8 * 4096, "partial-O staging fits the latent ring");
#pragma unroll 1
      for (int c = 0; c < kMlaHalf / 32; ++c) {
        uint32_t orr[32];
        if (nk > 0) {
          tmem_ld32(tmem + lane_base + kColO + c * 32, orr);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) orr[e] = 0u;
        }
        if (stage_o) {
          uint8_t* bx = sK + (warp * 8 + c) * 4096;
          const int lr = static_cast<int>(lane_id());
#pragma unroll
          for (int v = 0; v < 8; ++v)
            *reinterpret_cast<float4*>(bx + lr * 128 + ((v ^ (lr & 7)) << 4)) =
                make_float4(__uint_as_float(orr[v * 4]) * inv, __uint_as_float(orr[v * 4 + 1]) * inv,
                            __uint_as_float(orr[v * 4 + 2]) * inv,
                            __uint_as_float(orr[v * 4 + 3]) * inv);
          continue;
        }
        if (hh < p.heads) {
          float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
          for (int v = 0; v < 8; ++v)
            d4[v] = make_float4(__uint_as_float(orr[v * 4]) * inv, __uint_as_float(orr[v * 4 + 1]) * inv,
                                __uint_as_float(orr[v * 4 + 2]) * inv, __uint_as_float(orr[v * 4 + 3]) * inv);
        }
      }
      if (stage_o) {  // heads past p.heads are clipped by the map
        fence_proxy_async_smem();
        __syncwarp();
        if (lane_id() == 0) {
          for (int x = 0; x < 8; ++x)
            tma_store_4d(&tm_o, sK + (warp * 8 + x) * 4096, half * kMlaHalf + x * 32, warp * 32,
                         split, b);
          bulk_commit();
          bulk_wait<0>();
        }
      }
      if (half == 0 && hh < p.heads)
        p.part_lse[(static_cast<int64_t>(b) * p.splits + split) * p.heads + hh] = lse;
    } else {
      const bool live = i < p.seq_q;
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o) + b * p.o_sb + h * p.o_sh +
                            static_cast<int64_t>(live ? i : 0) * p.o_ss + half * kMlaHalf;
      // O through the (drained) latent ring as four SW128 [128][64] boxes and TMA stores
      const bool stage_o = p.o_tma != 0;
      static_assert(kSt * L::kKBytes >= 4 * 128 * 128, "O staging fits the latent ring");
#pragma unroll 1
      for (int c = 0; c < kMlaHalf / 32; ++c) {
        uint32_t orr[32];
        if (nk > 0) {
          tmem_ld32(tmem + lane_base + kColO + c * 32, orr);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) orr[e] = 0u;
        }
        if (stage_o) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int g = (c % 2) * 4 + v;
            *reinterpret_cast<uint4*>(sK + (c / 2) * (128 * 128) + row * 128 +
                                      ((g ^ (row & 7)) << 4)) = make_uint4(
                pack_bf16(__uint_as_float(orr[v * 8 + 0]) * inv, __uint_as_float(orr[v * 8 + 1]) * inv),
                pack_bf16(__uint_as_float(orr[v * 8 + 2]) * inv, __uint_as_float(orr[v * 8 + 3]) * inv),
                pack_bf16(__uint_as_float(orr[v * 8 + 4]) * inv, __uint_as_float(orr[v * 8 + 5]) * inv),
                pack_bf16(__uint_as_float(orr[v * 8 + 6]) * inv, __uint_as_float(orr[v * 8 + 7]) * inv));
          }
          continue;
        }
        if (live) {
          uint4* d4 = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            d4[v] = make_uint4(
                pack_bf16(__uint_as_float(orr[v * 8 + 0]) * inv, __uint_as_float(orr[v * 8 + 1]) * inv),
                pack_bf16(__uint_as_float(orr[v * 8 + 2]) * inv, __uint_as_float(orr[v * 8 + 3]) * inv),
                pack_bf16(__uint_as_float(orr[v * 8 + 4]) * inv, __uint_as_float(orr[v * 8 + 5]) * inv),
                pack_bf16(__uint_as_float(orr[v * 8 + 6]) * inv, __uint_as_float(orr[v * 8 + 7]) * inv));
        }
      }
      if (stage_o) {  // this warp's 32 rows of the four boxes (rows past seq_q are clipped)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane_id() == 0) {
#pragma unroll
          for (int x = 0; x < 4; ++x)
            tma_store_4d(&tm_o, sK + x * (128 * 128) + warp * 32 * 128, half * kMlaHalf + x * 64,
                         q0 + warp * 32, h, b);
          bulk_commit();
          bulk_wait<0>();
        }
      }
      if (half == 0 && live && p.lse != nullptr)
        p.lse[(static_cast<int64_t>(b) * p.heads + h) * p.seq_q + i] = lse;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Merge decode splits: O = sum_s e^{lse_s - lse} O_s, lse = log sum_s e^{lse_s}.
__global__ void mla_combine_kernel(const float* __restrict__ part_o,
                                   const float* __restrict__ part_lse, int batch, int heads,
                                   int splits, __nv_bfloat16* __restrict__ o,
                                   float* __restrict__ lse) {
  const int bh = blockIdx.x;  // one block per (b, head), 128 threads x 4 columns
  const int b = bh / heads, hh = bh % heads;
  float mx = -INFINITY;
  for (int s = 0; s < splits; ++s)
    mx = fmaxf(mx, part_lse[(static_cast<int64_t>(b) * splits + s) * heads + hh]);
  float den = 0.0f;
  for (int s = 0; s < splits; ++s) {
    const float l = part_lse[(static_cast<int64_t>(b) * splits + s) * heads + hh];
    den += (l == -INFINITY) ? 0.0f : __expf(l - mx);
  }
  const int c = threadIdx.x * 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < splits; ++s) {
    const float l = part_lse[(static_cast<int64_t>(b) * splits + s) * heads + hh];
    if (l == -INFINITY) continue;
    const float w = __expf(l - mx) / den;
    const float4 v = *reinterpret_cast<const float4*>(
        part_o + ((static_cast<int64_t>(b) * splits + s) * heads + hh) * kMlaDv + c);
    acc.x += w * v.x;
    acc.y += w * v.y;
    acc.z += w * v.z;
    acc.w += w * v.w;
  }
  uint2 out = make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
  *reinterpret_cast<uint2*>(o + (static_cast<int64_t>(b) * heads + hh) * kMlaDv + c) = out;
  if (threadIdx.x == 0 && lse != nullptr)
    lse[static_cast<int64_t>(b) * heads + hh] = (den == 0.0f) ? -INFINITY : mx + logf(den);
}

}  // namespace af
