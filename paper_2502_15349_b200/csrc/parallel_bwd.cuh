// K2 — parallel-template backward on sm_100a.
//
// Computes the VJP of K1 for a cotangent dO, i.e. what attnforge obtains by differentiating the
// dense pattern graph (attention.derive_backward, attention.py:529-550, adjoint rules
// graph.py:481-569) — restated in closed form:
//   softmax family     : P = exp(s - LSE), dV = P^T dO, dP = dO V^T, dS = P o (dP - D),
//                        D_i = sum_d dO_id O_id
//   elementwise family : P = act(z), dV = P^T dO, dP = dO V^T, dS = dP o act'(z) o mask
//   both               : dQ = tau dS K, dK = tau dS^T Q   (tau = q_mod scale)
// One CTA owns one 128-row key tile of one KV head and loops over every query head of its GQA
// group and every query tile the band mask lets it see, so dK/dV accumulate in TMEM and need no
// cross-CTA reduction.  dQ partial tiles are reduced into an fp32 accumulator in global memory.
//
// Warp roles (512 threads, <= 128 registers each):
//   warps 0-7  : key-row warps, two per TMEM lane quarter; warp w owns key row (w%4)*32+lane and
//                query columns [64*(w/4), 64*(w/4)+64): P^T, dS^T, then the dV (w<4) / dK store
//   warps 8-11 : dQ drain (TMEM -> registers, release TMEM, fp32 red.add into dq_accum)
//   warp  12   : TMA producer: K, V once; ring of (Q, dO, LSE, D) per query tile
//   warp  13   : TMEM allocator + tcgen05.mma issuer            (warps 14-15 idle)
// TMEM: [0,128) S^T -> P^T(bf16) | [128,256) dP^T -> dS^T(bf16) -> dQ | [256,256+DV) dV | dK
// Packed bf16 P^T / dS^T of query columns [0,64) land in packed columns [0,32) of their region
// and those of [64,128) in [64,96), so each warp only overwrites columns it alone has read.
#pragma once
#include <cuda.h>
#include "params.h"
#include "sm100.cuh"
#include "parallel_fwd.cuh"

namespace af {

#ifdef AF_TRACE
// Developer timeline of one CTA (blockIdx 0,0): g_af_trace[event][iteration] = clock64().
__device__ long long g_af_trace[16][512];
#define AF_T(ev, n)                                                              \
  do {                                                                           \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (n) < 512) g_af_trace[ev][n] = clock64(); \
  } while (0)
#else
#define AF_T(ev, n) \
  do {              \
  } while (0)
#endif

template <int D, int DV>
struct BwdSmem {
  static constexpr int kStages = 2;
  static constexpr int kKBytes = kBlockN * D * 2;
  static constexpr int kVBytes = kBlockN * DV * 2;
  static constexpr int kQBytes = kBlockM * D * 2;
  static constexpr int kOBytes = kBlockM * DV * 2;
  static constexpr int kKOff = 0;
  static constexpr int kVOff = kKOff + kKBytes;
  static constexpr int kQOff = kVOff + kVBytes;
  static constexpr int kOOff = kQOff + kStages * kQBytes;
  static constexpr int kDSOff = kOOff + kStages * kOBytes;
  static constexpr int kLseOff = kDSOff + kBlockM * kBlockN * 2;
  static constexpr int kDeltaOff = kLseOff + kStages * kBlockM * 4;
  static constexpr int kBarOff = kDeltaOff + kStages * kBlockM * 4;
  // kv_full, full[2], empty[2], s_full, dp_full, p_ready, ds_ready, dq_full, dq_free, acc_full
  static constexpr int kNumBars = 1 + 2 * kStages + 7;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
};

// Query-row range a key tile [k0, k0+128) is visible from under the band mask.
__host__ __device__ inline void query_band(const MaskParams& m, int k0, int seq_q, int& lo,
                                           int& hi) {
  lo = 0;
  hi = seq_q;
  if (m.causal) lo = max(0, k0 - m.diag_offset);
  if (m.window > 0) hi = min(seq_q, k0 + kBlockN - 1 - m.diag_offset + m.window);
}

AF_DEVICE bool block_fully_kept_t(const MaskParams& m, int q0, int k0, int seq_q, int seq_k) {
  if (q0 + kBlockM > seq_q) return false;
  return block_fully_kept(m, q0, k0, seq_k);
}

template <int kAct>
AF_DEVICE float act_grad(float z, float a) {  // a = act(z)
  if constexpr (kAct == kActSigmoid) {
    return a * (1.0f - a);
  } else if constexpr (kAct == kActRelu) {
    return z >= 0.0f ? 1.0f : 0.0f;  // ties route to the first max operand (graph.py:517-527)
  } else {
    return 1.0f;
  }
}

template <int D, int DV, int kFamily, int kAct>
__global__ void __launch_bounds__(512, 1)
    parallel_bwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                        const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v,
                        const __grid_constant__ CUtensorMap tm_do, const ParallelBwdParams p,
                        const float* __restrict__ lse2, const float* __restrict__ delta,
                        int seq_q_pad) {
  using L = BwdSmem<D, DV>;
  constexpr int kStages = L::kStages;
  static_assert(D % 64 == 0 && DV % 64 == 0 && D + DV <= 256, "tile dims");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sO = smem + L::kOOff;  // dO stages
  uint8_t* sDS = smem + L::kDSOff;
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
  uint64_t* dq_full = ds_ready + 1;
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
  const int qt_lo = qlo / kBlockM;
  const int qt_hi = (qhi > qlo) ? (qhi + kBlockM - 1) / kBlockM : qt_lo;
  const int tiles_per_head = qt_hi - qt_lo;
  const int niter = tiles_per_head * group;

  if (warp == 12 && lane_id() == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_ready, 8);
    mbar_init(ds_ready, 8);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 13) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + DV;
  // packed (bf16x2) column of the k-th 16-query slice of P^T / dS^T
  auto a_col = [](int kk) -> uint32_t { return kk < 4 ? kk * 8 : 64 + (kk - 4) * 8; };

  if (warp == 12) {
    // ───────────── TMA producer ─────────────
    if (elect_one() && niter > 0) {
      mbar_expect_tx(kv_full, L::kKBytes + L::kVBytes);
      for (int c = 0; c < D / 64; ++c)
        tma_load_4d(sK + c * (kBlockN * 128), &tm_k, kv_full, c * 64, k0, hk, b);
      for (int c = 0; c < DV / 64; ++c)
        tma_load_4d(sV + c * (kBlockN * 128), &tm_v, kv_full, c * 64, k0, hk, b);
      for (int n = 0; n < niter; ++n) {
        const int s = n % kStages;
        const uint32_t ph = (n / kStages) & 1;
        const int h = hk * group + n / tiles_per_head;
        const int q0 = (qt_lo + n % tiles_per_head) * kBlockM;
        mbar_wait(&empty[s], ph ^ 1);
        AF_T(10, n);
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
  } else if (warp == 13) {
    // ───────────── MMA issuer ─────────────
    if (elect_one() && niter > 0) {
      constexpr uint32_t id_s = make_idesc_bf16(kBlockN, kBlockM, false, false);   // S^T = K Q^T
      constexpr uint32_t id_dp = make_idesc_bf16(kBlockN, kBlockM, false, false);  // dP^T = V dO^T
      constexpr uint32_t id_dv = make_idesc_bf16(kBlockN, DV, false, true);        // dV += P^T dO
      constexpr uint32_t id_dk = make_idesc_bf16(kBlockN, D, false, true);         // dK += dS^T Q
      constexpr uint32_t id_dq = make_idesc_bf16(kBlockM, D, true, true);          // dQ = dS K
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ), aO = smem_u32(sO);
      const uint32_t aDS = smem_u32(sDS);
      auto kmajor = [](uint32_t base, int kk, int rows) {
        return make_sdesc(base + (kk / 4) * (rows * 128) + (kk % 4) * 32, 0, 1024);
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
      auto issue_dv = [&](int n) {  // dV += P^T dO  (A = P^T in TMEM, B = dO [q][dv] MN-major)
        const int s = n % kStages;
#pragma unroll
        for (int kk = 0; kk < kBlockM / 16; ++kk)
          mma_ts(tmem + kColDV, tmem + kColS + a_col(kk),
                 make_sdesc(aO + s * L::kOBytes + kk * 16 * 128, kBlockM * 128, 1024), id_dv,
                 (n > 0 || kk > 0));
      };
      auto wait_full = [&](int n) {
        mbar_wait(&full[n % kStages], (n / kStages) & 1);
        tc_fence_after();
      };
      // Issue order keeps the tensor pipe busy while the row warps and the dQ drain work:
      //   S0 dP0 | dV0 S1 | dK0 dQ0 | dV1 dP1 S2 | dK1 dQ1 | dV2 dP2 S3 | ...
      // TMEM reuse is safe because tcgen05.mma ops of one thread execute in issue order.
      mbar_wait(kv_full, 0);
      wait_full(0);
      issue_s(0);
      issue_dp(0);
      mbar_wait(p_ready, 0);
      tc_fence_after();
      issue_dv(0);
      if (niter > 1) {
        wait_full(1);
        issue_s(1);
      }
      for (int n = 0; n < niter; ++n) {
        const int s = n % kStages;
        // dK += dS^T Q ; dQ = dS K
        mbar_wait(ds_ready, n & 1);
        AF_T(0, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kBlockM / 16; ++kk)
          mma_ts(tmem + kColDK, tmem + kColDP + a_col(kk),
                 make_sdesc(aQ + s * L::kQBytes + kk * 16 * 128, kBlockM * 128, 1024), id_dk,
                 (n > 0 || kk > 0));
#pragma unroll
        for (int kk = 0; kk < kBlockN / 16; ++kk)
          mma_ss(tmem + kColDP, make_sdesc(aDS + kk * 16 * 128, kBlockN * 128, 1024),
                 make_sdesc(aK + kk * 16 * 128, kBlockN * 128, 1024), id_dq, kk > 0);
        mma_commit(dq_full);
        mma_commit(&empty[s]);
        if (n + 1 < niter) {
          mbar_wait(p_ready, (n + 1) & 1);
          AF_T(1, n + 1);
          tc_fence_after();
          issue_dv(n + 1);
          mbar_wait(dq_free, n & 1);
          AF_T(2, n + 1);
          tc_fence_after();
          issue_dp(n + 1);
          if (n + 2 < niter) {
            wait_full(n + 2);
            AF_T(3, n + 2);
            issue_s(n + 2);
          }
        }
      }
      mma_commit(acc_full);
    }
  } else if (warp < 8) {
    // ───────────── key-row warps ─────────────
    const int wq = warp % 4;
    const int half = warp / 4;
    const int row = wq * 32 + static_cast<int>(lane_id());
    const int j = k0 + row;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const int cb = half * 64;              // first query column owned by this warp
    const uint32_t pcol = half * 64;       // packed destination column (see header)
    const float fj = static_cast<float>(j);
    int hi_ = 0, qt_ = 0;                  // (query head, query tile) of iteration n
    for (int n = 0; n < niter; ++n) {
      const int s = n % kStages;
      const int h = hk * group + hi_;
      const int q0 = (qt_lo + qt_) * kBlockM;
      if (++qt_ == tiles_per_head) {
        qt_ = 0;
        ++hi_;
      }
      const bool fullblk = block_fully_kept_t(p.mask, q0, k0, p.seq_q, p.seq_k);
      float slope = 0.0f;
      if constexpr (kFamily == kFamilyElementwise) {
        if (p.slope != nullptr) slope = p.slope[h];
      }
      const float* lse_s = sLse + s * kBlockM + cb;
      const float* del_s = sDelta + s * kBlockM + cb;

      mbar_wait(s_full, n & 1);
      if (threadIdx.x == 0) AF_T(4, n);
      tc_fence_after();
      // P^T is kept as packed bf16 — exactly the operand the dV MMA consumes — and re-expanded
      // for dS; this halves the live registers of the row warps.
      uint32_t pk[32];
      uint32_t gmask[2];      // elementwise family: kept && act'(z) != 0 (relu / identity)
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        uint32_t sr[32];
        tmem_ld32(tmem + lane_base + kColS + cb + c2 * 32, sr);
        tmem_ld_wait();
        float pv[32];
        uint32_t bits = 0u;
        if constexpr (kFamily == kFamilySoftmax) {
          if (fullblk) {
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              const float4 l4 = *reinterpret_cast<const float4*>(lse_s + c2 * 32 + e);
              pv[e + 0] = ex2(fmaf(__uint_as_float(sr[e + 0]), p.scale_log2, -l4.x));
              pv[e + 1] = ex2(fmaf(__uint_as_float(sr[e + 1]), p.scale_log2, -l4.y));
              pv[e + 2] = ex2(fmaf(__uint_as_float(sr[e + 2]), p.scale_log2, -l4.z));
              pv[e + 3] = ex2(fmaf(__uint_as_float(sr[e + 3]), p.scale_log2, -l4.w));
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const int i = q0 + cb + c2 * 32 + e;
              const bool keep = kept(p.mask, i, j, p.seq_k) && i < p.seq_q;
              pv[e] = keep ? ex2(fmaf(__uint_as_float(sr[e]), p.scale_log2, -lse_s[c2 * 32 + e]))
                           : 0.0f;
            }
          }
        } else {
          const float zb = p.bias - slope * (static_cast<float>(q0 + cb + c2 * 32) - fj);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int i = q0 + cb + c2 * 32 + e;
            const float z = fmaf(__uint_as_float(sr[e]), p.scale, zb - slope * static_cast<float>(e));
            const bool keep = fullblk || (kept(p.mask, i, j, p.seq_k) && i < p.seq_q);
            const bool g = (kAct == kActRelu) ? (z >= 0.0f) : true;
            bits |= (keep && g) ? (1u << e) : 0u;
            pv[e] = keep ? apply_act<kAct>(z) : 0.0f;
          }
        }
        gmask[c2] = bits;
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[c2 * 16 + e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
      }
      tmem_st32(tmem + lane_base + kColS + pcol, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(p_ready);
      if (threadIdx.x == 0) AF_T(5, n);

      // dS^T = P^T o (dP^T - D)   |   dP^T o act'(z)
      mbar_wait(dp_full, n & 1);
      if (threadIdx.x == 0) AF_T(6, n);
      tc_fence_after();
      uint32_t dsk[32];
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        uint32_t dr[32];
        tmem_ld32(tmem + lane_base + kColDP + cb + c2 * 32, dr);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float p0 = __uint_as_float(pk[c2 * 16 + e / 2] << 16);
          const float p1 = __uint_as_float(pk[c2 * 16 + e / 2] & 0xFFFF0000u);
          const float p2 = __uint_as_float(pk[c2 * 16 + e / 2 + 1] << 16);
          const float p3 = __uint_as_float(pk[c2 * 16 + e / 2 + 1] & 0xFFFF0000u);
          float ds[4];
          if constexpr (kFamily == kFamilySoftmax) {
            const float4 d4 = *reinterpret_cast<const float4*>(del_s + c2 * 32 + e);
            ds[0] = p0 * (__uint_as_float(dr[e + 0]) - d4.x);
            ds[1] = p1 * (__uint_as_float(dr[e + 1]) - d4.y);
            ds[2] = p2 * (__uint_as_float(dr[e + 2]) - d4.z);
            ds[3] = p3 * (__uint_as_float(dr[e + 3]) - d4.w);
          } else if constexpr (kAct == kActSigmoid) {
            ds[0] = __uint_as_float(dr[e + 0]) * p0 * (1.0f - p0);
            ds[1] = __uint_as_float(dr[e + 1]) * p1 * (1.0f - p1);
            ds[2] = __uint_as_float(dr[e + 2]) * p2 * (1.0f - p2);
            ds[3] = __uint_as_float(dr[e + 3]) * p3 * (1.0f - p3);
          } else {
#pragma unroll
            for (int x = 0; x < 4; ++x)
              ds[x] = ((gmask[c2] >> (e + x)) & 1u) ? __uint_as_float(dr[e + x]) : 0.0f;
          }
          dsk[c2 * 16 + e / 2] = pack_bf16(ds[0], ds[1]);
          dsk[c2 * 16 + e / 2 + 1] = pack_bf16(ds[2], ds[3]);
        }
      }
      // dS^T into TMEM (A operand of dK) ...
      tmem_st32(tmem + lane_base + kColDP + pcol, dsk);
      // ... and into shared memory as the MN-major A operand of dQ = dS K: query chunk `half`
      // is [128 key rows][128 B] with 16-byte granules XOR-swizzled by (row % 8).
      if (n > 0) mbar_wait(dq_full, (n - 1) & 1);  // dQ_{n-1} finished reading sDS
      {
        uint8_t* base = sDS + half * (kBlockN * 128) + row * 128;
#pragma unroll
        for (int g = 0; g < 8; ++g)
          *reinterpret_cast<uint4*>(base + ((g ^ (row & 7)) * 16)) =
              make_uint4(dsk[g * 4 + 0], dsk[g * 4 + 1], dsk[g * 4 + 2], dsk[g * 4 + 3]);
      }
      fence_proxy_async_smem();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(ds_ready);
      if (threadIdx.x == 0) AF_T(7, n);
    }
    // ───────────── epilogue: warps 0-3 store dV, warps 4-7 store dK ─────────────
    if (niter > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
    }
    // Every lane runs the warp-collective TMEM loads; only rows inside seq_k store.
    const bool live = j < p.seq_k;
    const int ncol = half == 0 ? DV : D;
    const uint32_t col0 = half == 0 ? kColDV : kColDK;
    const float mul = half == 0 ? 1.0f : p.scale;
    __nv_bfloat16* dst =
        half == 0 ? reinterpret_cast<__nv_bfloat16*>(p.dv) + b * p.dv_stride_b +
                        hk * p.dv_stride_h + static_cast<int64_t>(live ? j : 0) * p.dv_stride_s
                  : reinterpret_cast<__nv_bfloat16*>(p.dk) + b * p.dk_stride_b +
                        hk * p.dk_stride_h + static_cast<int64_t>(live ? j : 0) * p.dk_stride_s;
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
      if (live) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(r[v * 8 + 0]) * mul, __uint_as_float(r[v * 8 + 1]) * mul);
          w.y = pack_bf16(__uint_as_float(r[v * 8 + 2]) * mul, __uint_as_float(r[v * 8 + 3]) * mul);
          w.z = pack_bf16(__uint_as_float(r[v * 8 + 4]) * mul, __uint_as_float(r[v * 8 + 5]) * mul);
          w.w = pack_bf16(__uint_as_float(r[v * 8 + 6]) * mul, __uint_as_float(r[v * 8 + 7]) * mul);
          d4[v] = w;
        }
      }
    }
  } else if (warp < 12) {
    // ───────────── dQ drain warps 8-11 ─────────────
    const int wq = warp % 4;
    const int row = wq * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    for (int n = 0; n < niter; ++n) {
      const int h = hk * group + n / tiles_per_head;
      const int q0 = (qt_lo + n % tiles_per_head) * kBlockM;
      mbar_wait(dq_full, n & 1);
      if (threadIdx.x == 256) AF_T(8, n);
      tc_fence_after();
      float* dst = p.dq_accum + ((static_cast<int64_t>(b) * p.heads_q + h) * seq_q_pad + q0 + row) * D;
      // Pull the tile out of TMEM in two 64-column halves; TMEM is released after the second
      // half lands, and the reductions of both halves are issued from registers.
      uint32_t r0[D / 2];
#pragma unroll
      for (int c = 0; c < D / 64; ++c)
        tmem_ld32(tmem + lane_base + kColDP + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&r0[c * 32]));
      tmem_ld_wait();
#ifndef AF_ABLATE_DQ_RED
#pragma unroll
      for (int v = 0; v < D / 8; ++v)
        atomicAdd(reinterpret_cast<float4*>(dst + v * 4),
                  make_float4(__uint_as_float(r0[v * 4]), __uint_as_float(r0[v * 4 + 1]),
                              __uint_as_float(r0[v * 4 + 2]), __uint_as_float(r0[v * 4 + 3])));
#endif
#pragma unroll
      for (int c = 0; c < D / 64; ++c)
        tmem_ld32(tmem + lane_base + kColDP + D / 2 + c * 32,
                  *reinterpret_cast<uint32_t(*)[32]>(&r0[c * 32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(dq_free);
      if (threadIdx.x == 256) AF_T(9, n);
#ifndef AF_ABLATE_DQ_RED
#pragma unroll
      for (int v = 0; v < D / 8; ++v)
        atomicAdd(reinterpret_cast<float4*>(dst + D / 2 + v * 4),
                  make_float4(__uint_as_float(r0[v * 4]), __uint_as_float(r0[v * 4 + 1]),
                              __uint_as_float(r0[v * 4 + 2]), __uint_as_float(r0[v * 4 + 3])));
#else
      if (r0[0] == 0x7fffffffu) dst[0] = 1.0f;  // keep the loads live
#endif
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// delta[b,h,i] = sum_d dO*O ; lse2 = LSE * log2(e) (padded rows: +inf -> P = 0, delta = 0)
template <int DV>
__global__ void bwd_preprocess_kernel(const __nv_bfloat16* __restrict__ o,
                                      const __nv_bfloat16* __restrict__ dout,
                                      const float* __restrict__ lse, int64_t o_sb, int64_t o_sh,
                                      int64_t o_ss, int64_t do_sb, int64_t do_sh, int64_t do_ss,
                                      int heads, int seq_q, int seq_q_pad, int family,
                                      float* __restrict__ lse2, float* __restrict__ delta,
                                      int64_t total_rows) {
  // one warp per query row
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t bh = gw / seq_q_pad;
  const int i = static_cast<int>(gw % seq_q_pad);
  if (gw >= total_rows) return;
  const int b = static_cast<int>(bh / heads), h = static_cast<int>(bh % heads);
  float acc = 0.0f;
  if (i < seq_q && family == kFamilySoftmax) {
    const __nv_bfloat16* orow = o + b * o_sb + h * o_sh + static_cast<int64_t>(i) * o_ss;
    const __nv_bfloat16* drow = dout + b * do_sb + h * do_sh + static_cast<int64_t>(i) * do_ss;
    for (int c = lane * 2; c < DV; c += 64) {
      const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(orow + c);
      const __nv_bfloat162 d = *reinterpret_cast<const __nv_bfloat162*>(drow + c);
      acc += __bfloat162float(a.x) * __bfloat162float(d.x) + __bfloat162float(a.y) * __bfloat162float(d.y);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    const int64_t idx = bh * seq_q_pad + i;
    delta[idx] = acc;
    float l = INFINITY;
    if (i < seq_q && family == kFamilySoftmax) {
      const float v = lse[(static_cast<int64_t>(b) * heads + h) * seq_q + i];
      l = (v == -INFINITY) ? INFINITY : v * kLog2e;  // fully-masked row: P = 0
    }
    lse2[idx] = l;
  }
}

// dq (bf16) = tau * dq_accum
template <int D>
__global__ void bwd_dq_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                                      int64_t sb, int64_t sh, int64_t ss, int heads, int seq_q,
                                      int seq_q_pad, float tau, int64_t total_rows) {
  const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t rowi = gt / (D / 8);
  const int c = static_cast<int>(gt % (D / 8)) * 8;
  if (rowi >= total_rows) return;
  const int64_t bh = rowi / seq_q;
  const int i = static_cast<int>(rowi % seq_q);
  const int b = static_cast<int>(bh / heads), h = static_cast<int>(bh % heads);
  const float4* src = reinterpret_cast<const float4*>(acc + (bh * seq_q_pad + i) * D + c);
  const float4 x = src[0], y = src[1];
  uint4 w;
  w.x = pack_bf16(x.x * tau, x.y * tau);
  w.y = pack_bf16(x.z * tau, x.w * tau);
  w.z = pack_bf16(y.x * tau, y.y * tau);
  w.w = pack_bf16(y.z * tau, y.w * tau);
  *reinterpret_cast<uint4*>(dq + b * sb + h * sh + static_cast<int64_t>(i) * ss + c) = w;
}

}  // namespace af
