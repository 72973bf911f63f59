// K2 — parallel-template backward on sm_100a: two atomic-free kernels.
//
// Computes the VJP of K1 for a cotangent dO, i.e. what attnforge obtains by differentiating the
// dense pattern graph (attention.derive_backward, attention.py:529-550; adjoint rules
// graph.py:481-569) — restated in closed form:
//   softmax family     : P = exp(s - LSE), dV = P^T dO, dP = dO V^T, dS = P o (dP - D),
//                        D_i = sum_d dO_id O_id
//   elementwise family : P = act(z), dV = P^T dO, dP = dO V^T, dS = dP o act'(z) o mask
//   both               : dQ = tau dS K, dK = tau dS^T Q   (tau = q_mod scale)
//
// K2a (key-tile stationary) accumulates dK, dV of one 128-row key tile in TMEM over every query
// head of its GQA group and every visible query tile: S^T = K Q^T, dP^T = V dO^T (SS MMAs),
// dV += P^T dO, dK += dS^T Q (A operand = packed bf16 P^T / dS^T straight from TMEM).
// K2b (query-tile stationary) accumulates dQ of one 128-row query tile in TMEM over the visible key
// tiles: S = Q K^T, dP = dO V^T, dQ += dS K, with Q and dO parked in TMEM as the A operands.
// No cross-CTA reduction exists, so results are bitwise deterministic (the reference's own
// determinism contract) at the price of recomputing S and dP in K2b.
//
// Both kernels: 320 threads.  warps 0-7 = row warps (two per TMEM lane quarter; warp w owns TMEM
// lane (w%4)*32+lane and columns [64*(w/4), 64*(w/4)+64) of the 128-wide score tile), warp 8 =
// TMA producer, warp 9 = TMEM allocator + single-thread tcgen05.mma issuer.
// Packed bf16 P / dS of score columns [0,64) land in packed columns [0,32) of their TMEM region
// and those of [64,128) in [64,96), so each warp only overwrites columns it alone has read.
#pragma once
#include <cuda.h>
#include "params.h"
#include "sm100.cuh"
#include "parallel_fwd.cuh"

namespace af {

// Developer timeline (-DAF_BWD_TRACE): SM-clock stamps of one K2b CTA, read back with
// af_debug_bwd_trace.  Compiled out of the product build.
#ifdef AF_BWD_TRACE
__device__ long long g_bwd_trace[10][256];
#define BWD_TRACE(ev, n)                                                                    \
  do {                                                                                      \
    if (blockIdx.x == 0 && blockIdx.y == 37 && lane_id() == 0 && (n) < 256)                \
      g_bwd_trace[ev][n] = clock64();                                                       \
  } while (0)
__device__ long long g_bwd2a_trace[6][512];
#define BWD2A_TRACE(ev, n)                                                                  \
  do {                                                                                      \
    if (blockIdx.x == 40 && blockIdx.y == 5 && lane_id() == 0 && (n) < 512)                \
      g_bwd2a_trace[ev][n] = clock64();                                                     \
  } while (0)
#else
#define BWD2A_TRACE(ev, n) \
  do {                     \
  } while (0)
#define BWD_TRACE(ev, n) \
  do {                   \
  } while (0)
#endif

#ifndef AF_BWD_POLY_MASK
#define AF_BWD_POLY_MASK 6  // fully-kept tiles: pairs with (e & mask) == 0 use exp2_poly (25 %; swept: 12.5 % 13.4 ms, 25 % 13.3 ms, 100 % 14.9 ms, none 14.0 ms)
#endif
// P recompute exponential: MUFU ex2, or the FMA-pipe polynomial for the selected pairs
AF_DEVICE float bwd_exp2(float x, int e) {
  if constexpr (AF_BWD_POLY_MASK >= 0) {
    if ((e & AF_BWD_POLY_MASK) == 0) return exp2_poly(x);
  }
  return ex2(x);
}

// packed (bf16x2) TMEM column of the k-th 16-wide K slice of a P / dS A operand
AF_DEVICE uint32_t split_col(int kk) { return kk < 4 ? kk * 8 : 64 + (kk - 4) * 8; }

// Query-row range a key tile [k0, k0+128) is visible from under the band mask.
__host__ __device__ inline void query_band(const MaskParams& m, int k0, int seq_q, int& lo,
                                           int& hi) {
  lo = 0;
  hi = seq_q;
  if (m.causal) lo = max(0, k0 - m.diag_offset);
  if (m.window > 0) hi = min(seq_q, k0 + kBlockN - 1 - m.diag_offset + m.window);
}

AF_DEVICE bool tile_fully_kept(const MaskParams& m, int q0, int k0, int seq_q, int seq_k) {
  if (q0 + kBlockM > seq_q) return false;
  return block_fully_kept(m, q0, k0, seq_k);
}

AF_DEVICE float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
AF_DEVICE float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

template <int N>
AF_DEVICE void store_row_bf16(__nv_bfloat16* dst, const uint32_t (&r)[N], float mul) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int v = 0; v < N / 8; ++v) {
    uint4 w;
    w.x = pack_bf16(__uint_as_float(r[v * 8 + 0]) * mul, __uint_as_float(r[v * 8 + 1]) * mul);
    w.y = pack_bf16(__uint_as_float(r[v * 8 + 2]) * mul, __uint_as_float(r[v * 8 + 3]) * mul);
    w.z = pack_bf16(__uint_as_float(r[v * 8 + 4]) * mul, __uint_as_float(r[v * 8 + 5]) * mul);
    w.w = pack_bf16(__uint_as_float(r[v * 8 + 6]) * mul, __uint_as_float(r[v * 8 + 7]) * mul);
    d4[v] = w;
  }
}

// dS from packed P and fp32 dP for NC (16 or 32) columns (both families)
// (soft-capped softmax: gk holds the packed factor cap_a cap_b (1 - t^2) of d s'/d s)
template <int kFamily, int kAct, bool kRowDelta, int NC = 32>
AF_DEVICE void make_ds(const uint32_t* pk, const uint32_t* dr, const float* del_col,
                       float del_row, uint32_t gmask, uint32_t* dsk, const uint32_t* gk) {
#pragma unroll
  for (int e = 0; e < NC; e += 2) {
    const uint32_t w = pk[e / 2];
    const float p0 = bf16_lo(w), p1 = bf16_hi(w);
    const float dp0 = __uint_as_float(dr[e]), dp1 = __uint_as_float(dr[e + 1]);
    float ds0, ds1;
    if constexpr (kFamily == kFamilySoftmax) {
      // ds = p (dP - delta): FADD2 + FMUL2 per pair
      const float2 t = fadd2(make_float2(dp0, dp1),
                             kRowDelta ? splat2(-del_row) : make_float2(-del_col[e], -del_col[e + 1]));
      const float2 d2 = fmul2(make_float2(p0, p1), t);
      ds0 = d2.x;
      ds1 = d2.y;
      if constexpr (kAct == kActSoftcap) {
        ds0 *= bf16_lo(gk[e / 2]);
        ds1 *= bf16_hi(gk[e / 2]);
      }
    } else if constexpr (kFamily == kFamilyAbssum) {
      // ds = (dP - [a >= 1] sign(s) D) / c, times the decay mask (gk = M / c); sign(0) = +1
      const float d0 = kRowDelta ? del_row : del_col[e];
      const float d1 = kRowDelta ? del_row : del_col[e + 1];
      ds0 = (dp0 - (((gmask >> e) & 1u) ? d0 : -d0)) * bf16_lo(gk[e / 2]);
      ds1 = (dp1 - (((gmask >> (e + 1)) & 1u) ? d1 : -d1)) * bf16_hi(gk[e / 2]);
    } else if constexpr (kAct == kActSigmoid) {
      ds0 = dp0 * p0 * (1.0f - p0);
      ds1 = dp1 * p1 * (1.0f - p1);
    } else if constexpr (kAct == kActRelu2) {  // d relu(z)^2 / dz = 2 relu(z) = 2 sqrt(p)
      ds0 = dp0 * 2.0f * sqrt_approx(p0);
      ds1 = dp1 * 2.0f * sqrt_approx(p1);
    } else {
      ds0 = ((gmask >> e) & 1u) ? dp0 : 0.0f;
      ds1 = ((gmask >> (e + 1)) & 1u) ? dp1 : 0.0f;
    }
    dsk[e / 2] = pack_bf16(ds0, ds1);
  }
}

// K2a / fused backward row math: P^T of one key row j against NC (16 or 32) consecutive query
// columns [i0, i0 + NC) from the raw scores sr (fp32 bits), packed bf16 into pk[NC/2]; gk[NC/2]
// receives the family's derivative factors (soft-cap, abssum); returns the keep /
// activation-gradient bits.
template <int kFamily, int kAct, int NC = 32>
AF_DEVICE uint32_t kv_rows_p32(const ParallelBwdParams& p, const uint32_t* sr, int i0, int j,
                               bool fullblk, float slope, const float* ls, uint32_t* pk,
                               uint32_t* gk) {
  uint32_t bits = 0u;
  // kept(i0 + c, j) & (i0 + c < seq_q) as one column range c in [c_lo, c_hi) for this key row:
  // two compares per element instead of kept()'s clamps (a key past seq_k keeps nothing);
  // evaluated only where a block is partial
  auto keep_at = [&](int c) {
    int c_lo = p.mask.causal ? j - p.mask.diag_offset - i0 : INT_MIN / 2;
    int c_hi = p.seq_q - i0;
    if (p.mask.window > 0) c_hi = min(c_hi, j - p.mask.diag_offset + p.mask.window - i0);
    if (j >= p.seq_k) c_lo = INT_MAX / 2;
    return fullblk | ((c >= c_lo) & (c < c_hi));
  };
  if constexpr (kFamily == kFamilySoftmax && kAct == kActSoftcap) {
    const float cap_in = p.cap_b * p.scale, cap_out = p.cap_a * kLog2e;
    const float cap_g = p.cap_a * p.cap_b;
#pragma unroll
    for (int e = 0; e < NC; e += 2) {
      float pv[2], gv[2];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int i = i0 + e + x;
        const bool keep = keep_at(e + x);
        const float t = tanh_precise(cap_in * __uint_as_float(sr[e + x]));
        pv[x] = keep ? ex2(fmaf(cap_out, t, -ls[e + x])) : 0.0f;
        gv[x] = cap_g * fmaf(-t, t, 1.0f);
      }
      pk[e / 2] = pack_bf16(pv[0], pv[1]);
      gk[e / 2] = pack_bf16(gv[0], gv[1]);
    }
  } else if constexpr (kFamily == kFamilyAbssum) {
    const bool norm = p.cap_a != 0.0f;
#pragma unroll
    for (int e = 0; e < NC; e += 2) {
      float pv[2], gv[2];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int i = i0 + e + x;
        const bool keep = keep_at(e + x);
        const float rc = norm ? rcp_approx(fmaxf(ls[e + x], 1.0f)) : 1.0f;
        const float m = ex2(static_cast<float>(i - j) * slope);
        const float z = __uint_as_float(sr[e + x]) * p.scale * m;
        pv[x] = keep ? z * rc : 0.0f;
        gv[x] = keep ? m * rc : 0.0f;
        bits |= (z >= 0.0f) ? (1u << (e + x)) : 0u;
      }
      pk[e / 2] = pack_bf16(pv[0], pv[1]);
      gk[e / 2] = pack_bf16(gv[0], gv[1]);
    }
  } else if constexpr (kFamily == kFamilySoftmax) {
    if (fullblk) {
#pragma unroll
      for (int e = 0; e < NC; e += 4) {
        // x = s * scale - lse: one FFMA2 per pair (the negation is an operand modifier)
        const float4 l4 = *reinterpret_cast<const float4*>(ls + e);
        const float2 sc2 = splat2(p.scale_log2);
        const float2 x01 =
            ffma2(make_float2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])), sc2,
                  make_float2(-l4.x, -l4.y));
        const float2 x23 =
            ffma2(make_float2(__uint_as_float(sr[e + 2]), __uint_as_float(sr[e + 3])), sc2,
                  make_float2(-l4.z, -l4.w));
        pk[e / 2] = pack_bf16(bwd_exp2(x01.x, e), bwd_exp2(x01.y, e));
        pk[e / 2 + 1] = pack_bf16(bwd_exp2(x23.x, e + 2), bwd_exp2(x23.y, e + 2));
      }
    } else {
#pragma unroll
      for (int e = 0; e < NC; e += 2) {
        float pv[2];
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const int i = i0 + e + x;
          const bool keep = keep_at(e + x);
          pv[x] = keep ? ex2(fmaf(__uint_as_float(sr[e + x]), p.scale_log2,
                                  -ls[e + x]))
                       : 0.0f;
        }
        pk[e / 2] = pack_bf16(pv[0], pv[1]);
      }
    }
  } else {
    const float zb = p.bias - slope * (static_cast<float>(i0) - static_cast<float>(j));
    if (fullblk) {  // compact fast path: no per-element mask tests
#pragma unroll
      for (int e = 0; e < NC; e += 2) {
        const float z0 = fmaf(__uint_as_float(sr[e]), p.scale, zb - slope * static_cast<float>(e));
        const float z1 = fmaf(__uint_as_float(sr[e + 1]), p.scale,
                              zb - slope * static_cast<float>(e + 1));
        if constexpr (kAct == kActRelu) {
          bits |= (z0 >= 0.0f ? (1u << e) : 0u) | (z1 >= 0.0f ? (2u << e) : 0u);
        } else {
          bits |= 3u << e;
        }
        pk[e / 2] = pack_bf16(apply_act<kAct>(z0), apply_act<kAct>(z1));
      }
    } else {
#pragma unroll  // fully: a partial unroll indexed pk through local memory
      for (int e = 0; e < NC; e += 2) {
        float pv[2];
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const int i = i0 + e + x;
          const float z = fmaf(__uint_as_float(sr[e + x]), p.scale,
                               zb - slope * static_cast<float>(e + x));
          const bool keep = keep_at(e + x);
          const bool g = (kAct == kActRelu) ? (z >= 0.0f) : true;
          bits |= (keep && g) ? (1u << (e + x)) : 0u;
          pv[x] = keep ? apply_act<kAct>(z) : 0.0f;
        }
        pk[e / 2] = pack_bf16(pv[0], pv[1]);
      }
    }
  }
  return bits;
}

// ═══════════════════════════════ K2a: dK, dV ═══════════════════════════════

// dS^T of K2a in shared memory instead of TMEM, so dP of the next tile can be issued ahead of dK:
// parity-green but measured slower (cfg2 bwd 12.6-12.9 -> 13.1-13.2 ms; tools/trace_bwd.py) —
// with one 32 KB buffer (no smem for two) the rows wait for dK of the previous tile before
// writing, which costs more than the earlier dP saves.  Off.
#ifndef AF_K2A_DS_SMEM
#define AF_K2A_DS_SMEM 0
#endif
template <int D, int DV>
struct BwdKVSmem {
  static constexpr int kStages = 2;
  static constexpr int kKBytes = kBlockN * D * 2;
  static constexpr int kVBytes = kBlockN * DV * 2;
  static constexpr int kQBytes = kBlockM * D * 2;
  static constexpr int kOBytes = kBlockM * DV * 2;
  static constexpr int kKOff = 0;
  static constexpr int kVOff = kKOff + kKBytes;
  static constexpr int kQOff = kVOff + kVBytes;
  static constexpr int kOOff = kQOff + kStages * kQBytes;
  static constexpr int kLseOff = kOOff + kStages * kOBytes;
  static constexpr int kDeltaOff = kLseOff + kStages * kBlockM * 4;
  // dS^T [128 keys][128 queries] bf16, K-major SW128 (A operand of dK += dS^T Q): kept in smem so
  // dP of the next tile can be issued before dK of this one (TMEM would alias it)
  static constexpr int kDsOff = AF_K2A_DS_SMEM ? ((kDeltaOff + kStages * kBlockM * 4 + 1023) & ~1023)
                                               : kDeltaOff + kStages * kBlockM * 4;
  static constexpr int kBarOff = kDsOff + (AF_K2A_DS_SMEM ? kBlockN * kBlockM * 2 : 0);
  // kv_full, full[S], empty[S], s_full, dp_full, p_ready, ds_ready, acc_full, ds_free
  static constexpr int kNumBars = 1 + 2 * kStages + 6;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
};

// K2a also runs 16 row warps (four per TMEM lane quarter, 32 query columns each).
constexpr int kKvRowWarps = 16;
constexpr int kKvThreads = 32 * (kKvRowWarps + 2);

template <int D, int DV, int kFamily, int kAct>
__global__ void __launch_bounds__(kKvThreads, 1)
    parallel_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_q,
                             const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v,
                             const __grid_constant__ CUtensorMap tm_do, const ParallelBwdParams p,
                             const float* __restrict__ lse2, const float* __restrict__ delta,
                             int seq_q_pad) {
  using L = BwdKVSmem<D, DV>;
  constexpr int kStages = L::kStages;
  static_assert(D % 64 == 0 && DV % 64 == 0 && D + DV <= 256, "tile dims");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sO = smem + L::kOOff;
  float* sLse = reinterpret_cast<float*>(smem + L::kLseOff);
  float* sDelta = reinterpret_cast<float*>(smem + L::kDeltaOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* kv_full = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + kStages;
  uint64_t* s_full = empty + kStages;
  uint64_t* dp_full = s_full + 1;
  uint64_t* p_ready = dp_full + 1;
  uint64_t* ds_ready = p_ready + 1;
  uint64_t* acc_full = ds_ready + 1;
  uint64_t* ds_free = acc_full + 1;  // dK of the previous tile has read sDS
  uint8_t* sDS = smem + L::kDsOff;
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
  const int qt_lo = qlo / kBlockM;
  const int qt_hi = (qhi > qlo) ? (qhi + kBlockM - 1) / kBlockM : qt_lo;
  const int tiles_per_head = qt_hi - qt_lo;
  const int niter = tiles_per_head * group;

  constexpr int kRW = kKvRowWarps, kTmaW = kRW, kMmaW = kRW + 1;
  constexpr int kCpw = kBlockM / (kRW / 4);  // query columns per row warp (32)
  constexpr int kNP = kCpw / 32;
  if (warp == kTmaW && lane_id() == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_ready, kRW);
    mbar_init(ds_ready, kRW);
    mbar_init(acc_full, 1);
    mbar_init(ds_free, 1);
    fence_barrier_init();
  }
  if (warp == kMmaW) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + DV;

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
        const int q0 = (qt_lo + qt_) * kBlockM;
        if (++qt_ == tiles_per_head) {
          qt_ = 0;
          ++hi_;
        }
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], L::kQBytes + L::kOBytes + 2 * kBlockM * 4);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d_hint(sQ + s * L::kQBytes + c * (kBlockM * 128), &tm_q, &full[s], c * 64, q0,
                           h, b, kEvictLast);
        for (int c = 0; c < DV / 64; ++c)
          tma_load_4d_hint(sO + s * L::kOBytes + c * (kBlockM * 128), &tm_do, &full[s], c * 64,
                           q0, h, b, kEvictLast);
        const int64_t row = (static_cast<int64_t>(b) * p.heads_q + h) * seq_q_pad + q0;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(sLse + s * kBlockM)),
            "l"(lse2 + row), "r"(kBlockM * 4), "r"(smem_u32(&full[s]))
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(sDelta + s * kBlockM)),
            "l"(delta + row), "r"(kBlockM * 4), "r"(smem_u32(&full[s]))
            : "memory");
      }
    }
  } else if (warp == kMmaW) {
    // ───────────── MMA issuer ─────────────
    if (elect_one() && niter > 0) {
      constexpr uint32_t id_s = make_idesc_bf16(kBlockN, kBlockM, false, false);   // S^T = K Q^T
      constexpr uint32_t id_dp = make_idesc_bf16(kBlockN, kBlockM, false, false);  // dP^T = V dO^T
      constexpr uint32_t id_dv = make_idesc_bf16(kBlockN, DV, false, true);        // dV += P^T dO
      constexpr uint32_t id_dk = make_idesc_bf16(kBlockN, D, false, true);         // dK += dS^T Q
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ), aO = smem_u32(sO);
      auto kmajor = [](uint32_t base, int kk, int rows) {
        return make_sdesc(base + (kk / 4) * (rows * 128) + (kk % 4) * 32, 0, 1024);
      };
      auto wait_full = [&](int n) {
        mbar_wait(&full[n % kStages], (n / kStages) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int n) {
        const int s = n % kStages;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem + kColS, kmajor(aK, kk, kBlockN), kmajor(aQ + s * L::kQBytes, kk, kBlockM),
                 id_s, kk > 0);
        mma_commit(s_full);
      };
      auto issue_dp = [&](int n) {
        const int s = n % kStages;
#pragma unroll
        for (int kk = 0; kk < DV / 16; ++kk)
          mma_ss(tmem + kColDP, kmajor(aV, kk, kBlockN), kmajor(aO + s * L::kOBytes, kk, kBlockM),
                 id_dp, kk > 0);
        mma_commit(dp_full);
      };
      // S0 dP0 | dV0 S1 | dK0 dP1 | dV1 S2 | dK1 dP2 | ...   (in-order tcgen05 execution makes
      // the TMEM reuse safe: S_{n+1} follows dV_n, which reads P^T_n; dP_{n+1} follows dK_n)
      mbar_wait(kv_full, 0);
      wait_full(0);
      issue_s(0);
      issue_dp(0);
      for (int n = 0; n < niter; ++n) {
        const int s = n % kStages;
        mbar_wait(p_ready, n & 1);
        BWD2A_TRACE(0, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kBlockM / 16; ++kk)
          mma_ts(tmem + kColDV, tmem + kColS + (kCpw * (kk / (kCpw / 16)) + 8 * (kk % (kCpw / 16))),
                 make_sdesc(aO + s * L::kOBytes + kk * 16 * 128, kBlockM * 128, 1024), id_dv,
                 (n > 0 || kk > 0));
        if (n + 1 < niter) {
          wait_full(n + 1);
          issue_s(n + 1);
        }
        mbar_wait(ds_ready, n & 1);
        BWD2A_TRACE(1, n);
        tc_fence_after();
        if constexpr (AF_K2A_DS_SMEM) {
          // dS^T lives in smem: dP of the next tile goes first (the row warps start on it while
          // the pipe runs dK of this tile)
          if (n + 1 < niter) issue_dp(n + 1);
          const uint32_t aDS = smem_u32(sDS);
#pragma unroll
          for (int kk = 0; kk < kBlockM / 16; ++kk)
            mma_ss(tmem + kColDK, kmajor(aDS, kk, kBlockN),
                   make_sdesc(aQ + s * L::kQBytes + kk * 16 * 128, kBlockM * 128, 1024), id_dk,
                   (n > 0 || kk > 0));
          mma_commit(ds_free);
          mma_commit(&empty[s]);
        } else {
#pragma unroll
          for (int kk = 0; kk < kBlockM / 16; ++kk)
            mma_ts(tmem + kColDK,
                   tmem + kColDP + (kCpw * (kk / (kCpw / 16)) + 8 * (kk % (kCpw / 16))),
                   make_sdesc(aQ + s * L::kQBytes + kk * 16 * 128, kBlockM * 128, 1024), id_dk,
                   (n > 0 || kk > 0));
          mma_commit(&empty[s]);
          if (n + 1 < niter) issue_dp(n + 1);
        }
      }
      mma_commit(acc_full);
    }
  } else {
    // ───────────── key-row warps ─────────────
    const int wq = warp % 4;
    const int sub = warp / 4;        // query-column slice of this warp
    const int row = wq * 32 + static_cast<int>(lane_id());
    const int j = k0 + row;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const int cb = sub * kCpw;
    const uint32_t pcol = cb;
    int slope_h = -1;
    float slope = 0.0f;
    int hi_ = 0, qt_ = 0;
    for (int n = 0; n < niter; ++n) {
      const int s = n % kStages;
      const int h = hk * group + hi_;
      const int q0 = (qt_lo + qt_) * kBlockM;
      if (++qt_ == tiles_per_head) {
        qt_ = 0;
        ++hi_;
      }
      const bool fullblk = tile_fully_kept(p.mask, q0, k0, p.seq_q, p.seq_k);
      if constexpr (kFamily != kFamilySoftmax) {  // once per head of the group
        if (h != slope_h) {
          slope_h = h;
          slope = p.slope != nullptr ? p.slope[h] : 0.0f;
        }
      }
      const float* lse_s = sLse + s * kBlockM + cb;
      const float* del_s = sDelta + s * kBlockM + cb;

      mbar_wait(s_full, n & 1);
      if (warp == 0) BWD2A_TRACE(2, n);
      tc_fence_after();
      uint32_t pk[16 * kNP];
      uint32_t gk[16 * kNP];  // soft-cap derivative factors (kActSoftcap only)
      uint32_t gmask[kNP];
#pragma unroll
      for (int c2 = 0; c2 < kNP; ++c2) {
        uint32_t sr[32];
        tmem_ld32(tmem + lane_base + kColS + cb + c2 * 32, sr);
        tmem_ld_wait();
        gmask[c2] = kv_rows_p32<kFamily, kAct>(p, sr, q0 + cb + c2 * 32, j, fullblk, slope,
                                               lse_s + c2 * 32, pk + c2 * 16, gk + c2 * 16);
      }
      if constexpr (kNP == 2)
        tmem_st32(tmem + lane_base + kColS + pcol, *reinterpret_cast<uint32_t(*)[32]>(pk));
      else
        tmem_st16(tmem + lane_base + kColS + pcol, *reinterpret_cast<uint32_t(*)[16]>(pk));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(p_ready);
      if (warp == 0) BWD2A_TRACE(3, n);

      mbar_wait(dp_full, n & 1);
      if (warp == 0) BWD2A_TRACE(4, n);
      tc_fence_after();
      uint32_t dsk[16 * kNP];
#pragma unroll
      for (int c2 = 0; c2 < kNP; ++c2) {
        uint32_t dr[32];
        tmem_ld32(tmem + lane_base + kColDP + cb + c2 * 32, dr);
        tmem_ld_wait();
        make_ds<kFamily, kAct, false>(pk + c2 * 16, dr, del_s + c2 * 32, 0.0f, gmask[c2],
                                      dsk + c2 * 16, gk + c2 * 16);
      }
      if constexpr (AF_K2A_DS_SMEM) {
        static_assert(kNP == 1, "dS^T smem slice is 32 query columns per warp");
        // this row's 32 query columns of dS^T: four 16-byte granules of the K-major SW128 tile
        if (n > 0) mbar_wait(ds_free, (n - 1) & 1);
        uint8_t* box = sDS + (cb / 64) * (kBlockN * 128);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int g = (cb % 64) / 8 + q;
          *reinterpret_cast<uint4*>(box + row * 128 + ((g ^ (row & 7)) << 4)) =
              make_uint4(dsk[q * 4], dsk[q * 4 + 1], dsk[q * 4 + 2], dsk[q * 4 + 3]);
        }
        fence_proxy_async_smem();
      } else {
        if constexpr (kNP == 2)
          tmem_st32(tmem + lane_base + kColDP + pcol, *reinterpret_cast<uint32_t(*)[32]>(dsk));
        else
          tmem_st16(tmem + lane_base + kColDP + pcol, *reinterpret_cast<uint32_t(*)[16]>(dsk));
        tmem_st_wait();
        tc_fence_before();
      }
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(ds_ready);
      if (warp == 0) BWD2A_TRACE(5, n);
    }
    // ───────────── epilogue: slices 0-1 store dV rows, slices 2-3 store dK rows ─────────────
    if (niter > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
    }
    const bool live = j < p.seq_k;
    const bool is_v = sub < (kRW / 8);
    const int part = is_v ? sub : sub - kRW / 8;  // which half of the dV / dK columns
    const int ncol = (is_v ? DV : D) / (kRW / 8);
    const uint32_t col0 = (is_v ? kColDV : kColDK) + part * ncol;
    const float mul = is_v ? 1.0f : p.scale;
    __nv_bfloat16* dst =
        (is_v ? reinterpret_cast<__nv_bfloat16*>(p.dv) + b * p.dv_stride_b +
                    hk * p.dv_stride_h + static_cast<int64_t>(live ? j : 0) * p.dv_stride_s
              : reinterpret_cast<__nv_bfloat16*>(p.dk) + b * p.dk_stride_b +
                    hk * p.dk_stride_h + static_cast<int64_t>(live ? j : 0) * p.dk_stride_s) +
        part * ncol;
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
      if (live) store_row_bf16<32>(dst + c * 32, r, mul);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaW) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ═══════════════════════════════ K2b: dQ ═══════════════════════════════

template <int D, int DV>
struct BwdQSmem {
  static constexpr int kStages = 3;
  static constexpr int kKBytes = kBlockN * D * 2;
  static constexpr int kVBytes = kBlockN * DV * 2;
  static constexpr int kKOff = 0;
  static constexpr int kVOff = kKOff + kStages * kKBytes;
  static constexpr int kBarOff = kVOff + kStages * kVBytes;
  // full[S], empty[S], qa_ready, s_full[2], dp_full[2], ds_ready[2], acc_full
  static constexpr int kNumBars = 2 * kStages + 8;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
};

// Load `W` packed bf16 words of one row (W*2 elements starting at src) into registers.
template <int W>
AF_DEVICE void load_row_words(const __nv_bfloat16* src, bool live, uint32_t (&w)[W]) {
#pragma unroll
  for (int v = 0; v < W / 4; ++v) {
    const uint4 x = live ? *reinterpret_cast<const uint4*>(src + v * 8) : make_uint4(0, 0, 0, 0);
    w[v * 4 + 0] = x.x;
    w[v * 4 + 1] = x.y;
    w[v * 4 + 2] = x.z;
    w[v * 4 + 3] = x.w;
  }
}

// K2b runs 16 row warps (four per TMEM lane quarter, 32 score columns each): its row math (P
// recompute + dS) is the critical path between the MMAs, and more warps hide the SFU latency.
constexpr int kDqRowWarps = 16;
constexpr int kDqThreads = 32 * (kDqRowWarps + 2);

template <int D, int DV, int kFamily, int kAct>
__global__ void __launch_bounds__(kDqThreads, 1)
    parallel_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const ParallelBwdParams p,
                           const __nv_bfloat16* __restrict__ q,
                           const __nv_bfloat16* __restrict__ dout, int64_t q_sb, int64_t q_sh,
                           int64_t q_ss, int64_t do_sb, int64_t do_sh, int64_t do_ss,
                           void* __restrict__ dq, const float* __restrict__ lse2,
                           const float* __restrict__ delta, int seq_q_pad) {
  using L = BwdQSmem<D, DV>;
  constexpr int kStages = L::kStages;
  static_assert(D % 64 == 0 && DV % 64 == 0 && D <= 128 && DV <= 128, "tile dims");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* qa_ready = empty + kStages;
  uint64_t* s_full = qa_ready + 1;   // [2]: one per 64-key column half
  uint64_t* dp_full = s_full + 2;    // [2]
  uint64_t* ds_ready = dp_full + 2;  // [2]
  uint64_t* acc_full = ds_ready + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);

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

  constexpr int kRW = kDqRowWarps, kTmaW = kRW, kMmaW = kRW + 1;
  constexpr int kCpw = kBlockN / (kRW / 4);  // score columns per row warp (32)
  // Row warps fetch their Q / dO slice and row statistics before the CTA set-up (barrier init,
  // TMEM allocation): the global-load latency hides behind it instead of following it.
  uint32_t qw[D / 8], ow[DV / 8];
  float l2 = INFINITY, dl = 0.0f;
  if (warp < kRW) {
    const int sub = warp / 4;
    const int i = q0 + (warp % 4) * 32 + static_cast<int>(lane_id());
    const bool live = i < p.seq_q;
    load_row_words<D / 8>(q + b * q_sb + h * q_sh + static_cast<int64_t>(live ? i : 0) * q_ss +
                              sub * (D / 4),
                          live, qw);
    load_row_words<DV / 8>(dout + b * do_sb + h * do_sh +
                               static_cast<int64_t>(live ? i : 0) * do_ss + sub * (DV / 4),
                           live, ow);
    const int64_t srow =
        (static_cast<int64_t>(b) * p.heads_q + h) * seq_q_pad + (live ? i : q0);
    if (live) {
      l2 = lse2[srow];  // +inf -> P = 0
      dl = delta[srow];
    }
  }
  if (warp == kTmaW && lane_id() == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(qa_ready, kRW);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&dp_full[x], 1);
      mbar_init(&ds_ready[x], kRW / 2);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == kMmaW) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // S [0,128) | dP [128,256) | dQ [256,256+D) | Q^A [384,384+D/2) | dO^A [448,448+DV/2)
  constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256, kColQA = 384, kColOA = 448;

  if (warp == kTmaW) {
    // ───────────── TMA producer: K/V ring ─────────────
    if (elect_one() && nk > 0) {
      for (int n = 0; n < nk; ++n) {
        const int s = n % kStages;
        const uint32_t ph = (n / kStages) & 1;
        const int kv0 = (band.jb_lo + n) * kBlockN;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], L::kKBytes + L::kVBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d_hint(sK + s * L::kKBytes + c * (kBlockN * 128), &tm_k, &full[s], c * 64,
                           kv0, hk, b, kEvictLast);
        for (int c = 0; c < DV / 64; ++c)
          tma_load_4d_hint(sV + s * L::kVBytes + c * (kBlockN * 128), &tm_v, &full[s], c * 64,
                           kv0, hk, b, kEvictLast);
      }
    }
  } else if (warp == kMmaW) {
    // ───────────── MMA issuer ─────────────
    if (elect_one() && nk > 0) {
      // The 128 key columns are processed as two 64-wide halves x = 0, 1 with their own
      // barriers: while the row warps of one half compute P / dS, the tensor pipe runs the other
      // half's dQ and the next tile's S / dP for the half already released (no TMEM to spare for
      // a second S/dP buffer, so the halves double-buffer each other).
      constexpr uint32_t id_s = make_idesc_bf16(kBlockM, kBlockN / 2, false, false);  // S = Q K^T
      constexpr uint32_t id_dq = make_idesc_bf16(kBlockM, D, false, true);            // dQ += dS K
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
      auto issue_sdp = [&](int n, int x) {
        const int s = n % kStages;
        const uint32_t kx = aK + s * L::kKBytes + x * 64 * 128;
        const uint32_t vx = aV + s * L::kVBytes + x * 64 * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ts(tmem + kColS + x * 64, tmem + kColQA + kk * 8,
                 make_sdesc(kx + (kk / 4) * (kBlockN * 128) + (kk % 4) * 32, 0, 1024), id_s,
                 kk > 0);
        mma_commit(&s_full[x]);
#pragma unroll
        for (int kk = 0; kk < DV / 16; ++kk)
          mma_ts(tmem + kColDP + x * 64, tmem + kColOA + kk * 8,
                 make_sdesc(vx + (kk / 4) * (kBlockN * 128) + (kk % 4) * 32, 0, 1024), id_s,
                 kk > 0);
        mma_commit(&dp_full[x]);
      };
      mbar_wait(qa_ready, 0);
      mbar_wait(&full[0], 0);
      tc_fence_after();
      issue_sdp(0, 0);
      issue_sdp(0, 1);
      for (int n = 0; n < nk; ++n) {
        const int s = n % kStages;
        const bool more = n + 1 < nk;
        for (int x = 0; x < 2; ++x) {
          mbar_wait(&ds_ready[x], n & 1);
          BWD_TRACE(x, n);
          tc_fence_after();
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int kk = x * 4 + k4;
            // packed dS of keys [16kk, 16kk + 16): the row warp owning those columns stored it
            // at the start of its own column range
            mma_ts(tmem + kColDQ, tmem + kColS + kCpw * (kk / (kCpw / 16)) + 8 * (kk % (kCpw / 16)),
                   make_sdesc(aK + s * L::kKBytes + kk * 16 * 128, kBlockN * 128, 1024), id_dq,
                   (n > 0 || kk > 0));
          }
          if (x == 1) mma_commit(&empty[s]);
          if (more) {
            if (x == 0) {
              mbar_wait(&full[(n + 1) % kStages], ((n + 1) / kStages) & 1);
              tc_fence_after();
            }
            issue_sdp(n + 1, x);
            BWD_TRACE(2 + x, n);
          }
        }
      }
      mma_commit(acc_full);
    }
  } else {
    // ───────────── query-row warps ─────────────
    const int wq = warp % 4;
    const int sub = warp / 4;              // column slice of this warp
    const int cb = sub * kCpw;
    const int half = cb / 64;              // MMA column half it belongs to
    const int row = wq * 32 + static_cast<int>(lane_id());
    const int i = q0 + row;
    const bool live = i < p.seq_q;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t pcol = cb;
    constexpr int kNP = kCpw / 32;         // 32-column pieces per warp
    // Park this row's Q and dO (bf16) in TMEM as the K-major A operands: the four warps of a
    // lane quarter each write a quarter of the packed words (D/8 of Q^A, DV/8 of dO^A).
    {
      static_assert(kRW == 16, "parking split assumes four warps per lane quarter");
      if constexpr (D == 128)
        tmem_st16(tmem + lane_base + kColQA + sub * 16, qw);
      else
        tmem_st8(tmem + lane_base + kColQA + sub * 8, qw);
      if constexpr (DV == 128)
        tmem_st16(tmem + lane_base + kColOA + sub * 16, ow);
      else
        tmem_st8(tmem + lane_base + kColOA + sub * 8, ow);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(qa_ready);
    }
    float slope = 0.0f;
    if constexpr (kFamily != kFamilySoftmax) {
      if (p.slope != nullptr) slope = p.slope[h];
    }
    const float fi = static_cast<float>(i);
    for (int n = 0; n < nk; ++n) {
      const int c0 = (band.jb_lo + n) * kBlockN;
      const bool fullblk = tile_fully_kept(p.mask, q0, c0, p.seq_q, p.seq_k);
      mbar_wait(&s_full[half], n & 1);
      if (warp % 8 == 0) BWD_TRACE(4 + half, n);
      tc_fence_after();
      uint32_t pk[16 * kNP];
      uint32_t gk[16 * kNP];  // soft-cap derivative factors (kActSoftcap only)
      uint32_t gmask[kNP];
#pragma unroll
      for (int c2 = 0; c2 < kNP; ++c2) {
        uint32_t sr[32];
        tmem_ld32(tmem + lane_base + kColS + cb + c2 * 32, sr);
        tmem_ld_wait();
        uint32_t bits = 0u;
        const int jb = c0 + cb + c2 * 32;
        if constexpr (kFamily == kFamilySoftmax && kAct == kActSoftcap) {
          const float cap_in = p.cap_b * p.scale, cap_out = p.cap_a * kLog2e;
          const float cap_g = p.cap_a * p.cap_b;
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float pv[2], gv[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) {
              const bool keep = fullblk | kept(p.mask, i, jb + e + x, p.seq_k);
              const float t = tanh_precise(cap_in * __uint_as_float(sr[e + x]));
              pv[x] = keep ? ex2(fmaf(cap_out, t, -l2)) : 0.0f;
              gv[x] = cap_g * fmaf(-t, t, 1.0f);
            }
            pk[c2 * 16 + e / 2] = pack_bf16(pv[0], pv[1]);
            gk[c2 * 16 + e / 2] = pack_bf16(gv[0], gv[1]);
          }
        } else if constexpr (kFamily == kFamilyAbssum) {
          const float rc = (p.cap_a != 0.0f) ? rcp_approx(fmaxf(l2, 1.0f)) : 1.0f;
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float pv[2], gv[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) {
              const int jj = jb + e + x;
              const bool keep = live & (fullblk | kept(p.mask, i, jj, p.seq_k));
              const float m = ex2(static_cast<float>(i - jj) * slope);
              const float z = __uint_as_float(sr[e + x]) * p.scale * m;
              pv[x] = keep ? z * rc : 0.0f;
              gv[x] = keep ? m * rc : 0.0f;
              bits |= (z >= 0.0f) ? (1u << (e + x)) : 0u;
            }
            pk[c2 * 16 + e / 2] = pack_bf16(pv[0], pv[1]);
            gk[c2 * 16 + e / 2] = pack_bf16(gv[0], gv[1]);
          }
        } else if constexpr (kFamily == kFamilySoftmax) {
          if (fullblk) {
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const float2 x = ffma2(make_float2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])),
                                     splat2(p.scale_log2), splat2(-l2));
              pk[c2 * 16 + e / 2] = pack_bf16(bwd_exp2(x.x, e), bwd_exp2(x.y, e));
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const bool a0 = kept(p.mask, i, jb + e, p.seq_k);
              const bool a1 = kept(p.mask, i, jb + e + 1, p.seq_k);
              pk[c2 * 16 + e / 2] =
                  pack_bf16(a0 ? ex2(fmaf(__uint_as_float(sr[e]), p.scale_log2, -l2)) : 0.0f,
                            a1 ? ex2(fmaf(__uint_as_float(sr[e + 1]), p.scale_log2, -l2)) : 0.0f);
            }
          }
        } else {
          const float zb = p.bias - slope * (fi - static_cast<float>(jb));
          if (fullblk && live) {  // compact fast path: no per-element mask tests
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const float z0 = fmaf(__uint_as_float(sr[e]), p.scale, zb + slope * static_cast<float>(e));
              const float z1 = fmaf(__uint_as_float(sr[e + 1]), p.scale,
                                    zb + slope * static_cast<float>(e + 1));
              if constexpr (kAct == kActRelu) {
                bits |= (z0 >= 0.0f ? (1u << e) : 0u) | (z1 >= 0.0f ? (2u << e) : 0u);
              } else {
                bits |= 3u << e;
              }
              pk[c2 * 16 + e / 2] = pack_bf16(apply_act<kAct>(z0), apply_act<kAct>(z1));
            }
          } else {
#pragma unroll  // fully: a partial unroll indexed pk through local memory
            for (int e = 0; e < 32; e += 2) {
              float pv[2];
#pragma unroll
              for (int x = 0; x < 2; ++x) {
                const float z = fmaf(__uint_as_float(sr[e + x]), p.scale,
                                     zb + slope * static_cast<float>(e + x));
                const bool keep = live & kept(p.mask, i, jb + e + x, p.seq_k);
                const bool g = (kAct == kActRelu) ? (z >= 0.0f) : true;
                bits |= (keep && g) ? (1u << (e + x)) : 0u;
                pv[x] = keep ? apply_act<kAct>(z) : 0.0f;
              }
              pk[c2 * 16 + e / 2] = pack_bf16(pv[0], pv[1]);
            }
          }
        }
        gmask[c2] = bits;
      }
      mbar_wait(&dp_full[half], n & 1);
      if (warp % 8 == 0) BWD_TRACE(6 + half, n);
      tc_fence_after();
      uint32_t dsk[16 * kNP];
#pragma unroll
      for (int c2 = 0; c2 < kNP; ++c2) {
        uint32_t dr[32];
        tmem_ld32(tmem + lane_base + kColDP + cb + c2 * 32, dr);
        tmem_ld_wait();
        make_ds<kFamily, kAct, true>(pk + c2 * 16, dr, nullptr, dl, gmask[c2], dsk + c2 * 16,
                                     gk + c2 * 16);
      }
      // dS (packed) over this warp's own S columns: A operand of dQ += dS K
      if constexpr (kNP == 2)
        tmem_st32(tmem + lane_base + kColS + pcol, *reinterpret_cast<uint32_t(*)[32]>(dsk));
      else
        tmem_st16(tmem + lane_base + kColS + pcol, *reinterpret_cast<uint32_t(*)[16]>(dsk));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&ds_ready[half]);
      if (warp % 8 == 0) BWD_TRACE(8 + half, n);
    }
    // ───────────── epilogue: dQ = tau * acc (bf16); each warp stores D/4 columns ─────────────
    if (nk > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
    }
    __nv_bfloat16* dqrow = reinterpret_cast<__nv_bfloat16*>(dq) + b * q_sb + h * q_sh +
                           static_cast<int64_t>(live ? i : 0) * q_ss + sub * (D / 4);
    if constexpr (D / 4 == 32) {
      uint32_t r[32];
      if (nk > 0) {
        tmem_ld32(tmem + lane_base + kColDQ + sub * 32, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) r[e] = 0u;
      }
      if (live) store_row_bf16<32>(dqrow, r, p.scale);
    } else {
      static_assert(D / 4 == 16, "dQ epilogue slice");
      uint32_t r[16];
      if (nk > 0) {
        tmem_ld16(tmem + lane_base + kColDQ + sub * 16, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] = 0u;
      }
      if (live) store_row_bf16<16>(dqrow, r, p.scale);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaW) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// delta[b,h,i] = sum_d dO*O ; lse2 = LSE * log2(e) (padded / fully-masked rows: +inf -> P = 0)
// DV / 32 threads per row, each streaming 32 columns of O and dO as four 16-byte vectors (eight
// loads in flight per thread; a warp-per-row form with 4-byte loads ran at 0.30 of HBM).
template <int DV>
__global__ void __launch_bounds__(256) bwd_preprocess_kernel(
    const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, int64_t o_sb, int64_t o_sh, int64_t o_ss, int64_t do_sb,
    int64_t do_sh, int64_t do_ss, int heads, int seq_q, int seq_q_pad, int family,
    float* __restrict__ lse2, float* __restrict__ delta, int64_t total_rows,
    float* __restrict__ dq_zero = nullptr) {
  constexpr int kTpr = DV / 32;  // threads per row
  static_assert(kTpr >= 1 && kTpr <= 32 && (kTpr & (kTpr - 1)) == 0, "DV");
  const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t gw = gt / kTpr;  // row
  const int part = static_cast<int>(gt % kTpr);
  const bool row_ok = gw < total_rows;
  const int64_t row = row_ok ? gw : 0;
  const int64_t bh = row / seq_q_pad;
  const int i = static_cast<int>(row % seq_q_pad);
  const int b = static_cast<int>(bh / heads), h = static_cast<int>(bh % heads);
  float acc = 0.0f;
  // family 2 = abssum (normalised rows), 3 = abssum without the row norm (internal codes)
  const bool need_d = family == kFamilySoftmax || family == 2;
  if (row_ok && i < seq_q && need_d) {
    const uint4* orow = reinterpret_cast<const uint4*>(
        o + b * o_sb + h * o_sh + static_cast<int64_t>(i) * o_ss + part * 32);
    const uint4* drow = reinterpret_cast<const uint4*>(
        dout + b * do_sb + h * do_sh + static_cast<int64_t>(i) * do_ss + part * 32);
    uint4 ov[4], dv[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      ov[v] = __ldg(orow + v);
      dv[v] = __ldg(drow + v);
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint32_t* oe = reinterpret_cast<const uint32_t*>(&ov[v]);
      const uint32_t* de = reinterpret_cast<const uint32_t*>(&dv[v]);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        acc += bf16_lo_(oe[e]) * bf16_lo_(de[e]) + bf16_hi_(oe[e]) * bf16_hi_(de[e]);
    }
  }
  // the fused backward's fp32 dQ accumulator (dq_accum_offset layout, Dqk = DV = 128: one 32-col
  // chunk per thread) is zeroed here rather than by a separate memset pass
  // (a 256-thread block covers 64 rows = one 64-row query tile of one head, whose accumulator
  // tile is 32 KB contiguous: written as coalesced float4 sweeps)
  if (kTpr == 4 && dq_zero != nullptr && static_cast<int64_t>(blockIdx.x) * 64 < total_rows) {
    float4* z = reinterpret_cast<float4*>(dq_zero) + static_cast<int64_t>(blockIdx.x) * 2048;
#pragma unroll
    for (int v = 0; v < 8; ++v) z[v * 256 + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int off = kTpr / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (row_ok && part == 0) {
    float l = INFINITY;
    if (family == kFamilySoftmax) {
      if (i < seq_q) {
        const float v = lse[(static_cast<int64_t>(b) * heads + h) * seq_q + i];
        l = (v == -INFINITY) ? INFINITY : v * kLog2e;  // fully-masked row: P = 0
      }
    } else if (family == 2 || family == 3) {  // row abs-sum a_i; D only where the clamp is off
      const float a = (i < seq_q) ? lse[(static_cast<int64_t>(b) * heads + h) * seq_q + i] : 0.0f;
      l = (i < seq_q) ? a : INFINITY;
      if (family == 3 || a < 1.0f) acc = 0.0f;
    }
    delta[gw] = acc;
    lse2[gw] = l;
  }
}

}  // namespace af
