// K4w — linear (recurrent) template, one CTA per (b, h) over the whole 128-wide value dimension
// (Dk = Dv = 128), sm_100a.
//
// Same recurrence and chunk decomposition as linear_chunk_kernel (linear_chunk.cuh: engine.py
// run_step_recurrent / run_chunk_recurrent, engine.py:525-616), per chunk of C = 128:
//   forward : O_c = s_out [ ((Q K^T) o D) V + (Q o cp) H_in ],  H_out = g H_in + (K o w)^T V
//             D[i,u] = 2^{l_i - l_u} u_u [u <= i], cp_i = 2^{l_i}, w_u = u_u 2^{l_last - l_u}
//   reverse : D[i,u] = 2^{l_u - l_i} u_u [u >= i], cp_i = 2^{l_last - l_i}, w_u = u_u 2^{l_u},
//             chunks last to first (l = in-chunk inclusive cumsum of log2 a, g = 2^{l_last})
// but with the whole value dimension in one CTA, so S = Q K^T is computed once per chunk instead
// of once per 64-column value slice, and every GEMM is 128 x 128 x 128 (N = 64 tcgen05.mma runs at
// two thirds of its floor, tools/micro/mma_rate.cu).  The 64-column kernel spends a 4.2k-clk
// chunk period (tools/trace_linear.py, cfg5b) on 1.7k clk of MMA with its row warps' shared-memory
// accesses queued behind the SS GEMMs' operand reads; here the per-chunk work is
//   S = Q K^T (SS) | O = Q Hb (SS, Hb = bf16 copy of H_in) | H = g H + Kw^T V (SS, Kw = diag(w) K
//   scaled in place once S has read K) | O += P V (TS, P = S o D packed bf16 in the S columns)
// with the row warps scaling the Q Hb rows by cp_i in TMEM before P V accumulates onto them.
//   warps 0-7   chunk-row warps (two per TMEM lane quarter, key / column halves): P, Kw, cp-scale
//   warps 8-11  state warps (TMEM lane = d_k row): Hb copy, H *= g of the next chunk, final state
//   warps 12-15 output warps: O (double-buffered in TMEM) -> bf16 rows (+ the optional dot)
//   warp 16     TMA producer (Q/K/V ring of 2; the chunk's scan arrays with the same barrier)
//   warp 17     TMEM allocator + single-thread tcgen05.mma issuer
// TMEM: S / P [0,128) | O x2 [128,384) | H [384,512).
#pragma once
#include <cuda.h>
#include "params.h"
#include "sm100.cuh"
#include "linear_chunk.cuh"

namespace af {

struct LinWideSmem {
  static constexpr int kStages = 2;
  static constexpr int kTile = kLinChunk * 128 * 2;  // 128 x 128 bf16 (two 64-column SW128 boxes)
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + kStages * kTile;
  static constexpr int kVOff = kKOff + kStages * kTile;
  static constexpr int kHbOff = kVOff + kStages * kTile;
  static constexpr int kLOff = kHbOff + kTile;                 // [2][128] in-chunk cumsum log2 a
  static constexpr int kUOff = kLOff + kStages * kLinChunk * 4;  // [2][128] key-side scale
  static constexpr int kBarOff = kUOff + kStages * kLinChunk * 4;
  // full[2] (Q + scan arrays), empty[2] (Q), kfull[2], kempty[2], vfull[2], vempty[2], s_full,
  // qh_full, pk_ready, o_scaled, h_full, hb_ready, h_scaled, oi_full[2], o_empty[2]
  static constexpr int kNumBars = 6 * kStages + 7 + 4;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  // separable decay: per-chunk column factors b_u and the row warps' deviation maxima
  static constexpr int kBOff = (kTmemSlotOff + 16 + 15) / 16 * 16;  // [128] fp32, 16-B aligned
  static constexpr int kDevOff = kBOff + kLinChunk * 4;      // [4] fp32
  static constexpr int kTotal = kDevOff + 16;
};
static_assert(LinWideSmem::kTotal <= 232448, "wide linear kernel: shared memory");

constexpr int kLinWideThreads = 18 * 32;

template <bool kReverse>
__global__ void __launch_bounds__(kLinWideThreads, 1)
    linear_wide_kernel(const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const LinearParams p) {
  using L = LinWideSmem;
  constexpr int kSt = L::kStages;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint8_t* sHb = smem + L::kHbOff;
  float* sL = reinterpret_cast<float*>(smem + L::kLOff);
  float* sU = reinterpret_cast<float*>(smem + L::kUOff);
  float* sB = reinterpret_cast<float*>(smem + L::kBOff);
  float* sDev = reinterpret_cast<float*>(smem + L::kDevOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  // Q, K and V rings with their own barriers, each slot released by its last reader (Q after
  // Q Hb, K after the state update, V after P V) so the next loads start as early as possible
  // (the kernel streams 128 KB per chunk and SM; one shared slot release after P V left the loads
  // a chunk period behind)
  uint64_t* full = bars;            // Q + the chunk's scan arrays
  uint64_t* empty = full + kSt;
  uint64_t* kfull = empty + kSt;
  uint64_t* kempty = kfull + kSt;
  uint64_t* vfull = kempty + kSt;
  uint64_t* vempty = vfull + kSt;
  uint64_t* s_full = vempty + kSt;
  uint64_t* qh_full = s_full + 1;
  uint64_t* pk_ready = qh_full + 1;   // P in TMEM and Kw in smem (8 row warps)
  uint64_t* o_scaled = pk_ready + 1;  // Q Hb rows scaled by cp (8 row warps)
  uint64_t* h_full = o_scaled + 1;
  uint64_t* hb_ready = h_full + 1;    // Hb = bf16(H) written (4 state warps)
  uint64_t* h_scaled = hb_ready + 1;  // H *= g of the next chunk (4 state warps)
  uint64_t* oi_full = h_scaled + 1;   // [2]
  uint64_t* o_empty = oi_full + 2;    // [2] (4 output warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);

  const int warp = static_cast<int>(warp_id());
  const int bh = blockIdx.x;
  const int b = bh / p.heads;
  const int h = bh % p.heads;
  const int nchunks = (p.seq + kLinChunk - 1) / kLinChunk;
  constexpr int kTmaW = 16, kMmaW = 17;

  if (warp == kTmaW && lane_id() == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&kfull[s], 1);
      mbar_init(&kempty[s], 1);
      mbar_init(&vfull[s], 1);
      mbar_init(&vempty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(qh_full, 1);
    mbar_init(pk_ready, 8);
    mbar_init(o_scaled, 8);
    mbar_init(h_full, 1);
    mbar_init(hb_ready, 4);
    mbar_init(h_scaled, 4);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&oi_full[x], 1);
      mbar_init(&o_empty[x], 4);
    }
    fence_barrier_init();
  }
  if (warp == kMmaW) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kColS = 0, kColO = 128, kColH = 384;
  auto chunk_of = [&](int n) { return kReverse ? nchunks - 1 - n : n; };

  if (warp == kTmaW) {
    // ───────────── TMA producer: Q, K, V and the chunk's scan arrays ─────────────
    if (elect_one()) {
      for (int n = 0; n < nchunks; ++n) {
        const int s = n % kSt;
        const int c = chunk_of(n);
        const int t0 = c * kLinChunk;
        const uint32_t ph = ((n / kSt) & 1) ^ 1;
        mbar_wait(&empty[s], ph);
        AF_LT(15, n);
        const int64_t g = (static_cast<int64_t>(bh) * nchunks + c) * kLinChunk;
        const uint32_t scan_bytes = kLinChunk * 4 * (p.ucum != nullptr ? 2 : 1);
        mbar_expect_tx(&full[s], L::kTile + scan_bytes);
        for (int x = 0; x < 2; ++x)
          tma_load_4d(sQ + s * L::kTile + x * (kLinChunk * 128), &tm_q, &full[s], x * 64, t0, h,
                      b);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(sL + s * kLinChunk)),
            "l"(p.lcum + g), "r"(kLinChunk * 4), "r"(smem_u32(&full[s]))
            : "memory");
        if (p.ucum != nullptr)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
              "[%3];" ::"r"(smem_u32(sU + s * kLinChunk)),
              "l"(p.ucum + g), "r"(kLinChunk * 4), "r"(smem_u32(&full[s]))
              : "memory");
        mbar_wait(&kempty[s], ph);
        mbar_expect_tx(&kfull[s], L::kTile);
        for (int x = 0; x < 2; ++x)
          tma_load_4d(sK + s * L::kTile + x * (kLinChunk * 128), &tm_k, &kfull[s], x * 64, t0, h,
                      b);
        mbar_wait(&vempty[s], ph);
        mbar_expect_tx(&vfull[s], L::kTile);
        for (int x = 0; x < 2; ++x)
          tma_load_4d(sV + s * L::kTile + x * (kLinChunk * 128), &tm_v, &vfull[s], x * 64, t0, h,
                      b);
      }
    }
  } else if (warp == kMmaW) {
    // ───────────── MMA issuer: S | Q Hb | H update | P V ─────────────
    if (elect_one()) {
      constexpr uint32_t id_s = make_idesc_bf16(128, 128, false, false);  // S = Q K^T
      constexpr uint32_t id_qh = make_idesc_bf16(128, 128, false, true);  // O = Q Hb
      constexpr uint32_t id_h = make_idesc_bf16(128, 128, true, true);    // H += Kw^T V
      constexpr uint32_t id_oi = make_idesc_bf16(128, 128, false, true);  // O += P V
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV), aHb = smem_u32(sHb);
      auto kmaj = [](uint32_t base, int kk) {
        return make_sdesc(base + (kk / 4) * (kLinChunk * 128) + (kk % 4) * 32, 0, 1024);
      };
      for (int n = 0; n < nchunks; ++n) {
        const int s = n % kSt;
        const uint32_t ob = n & 1;
        const uint32_t qa = aQ + s * L::kTile, ka = aK + s * L::kTile, va = aV + s * L::kTile;
        const uint32_t o_tmem = tmem + kColO + ob * 128;
        mbar_wait(&full[s], (n / kSt) & 1);
        mbar_wait(&kfull[s], (n / kSt) & 1);
        AF_LT(0, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ss(tmem + kColS, kmaj(qa, kk), kmaj(ka, kk), id_s, kk > 0);
        mma_commit(s_full);
        if (n >= 2) mbar_wait(&o_empty[ob], ((n >> 1) - 1) & 1);  // chunk n-2's output drained
        if (n > 0) {
          mbar_wait(hb_ready, (n - 1) & 1);  // Hb = H after chunk n-1
          AF_LT(1, n);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ss(o_tmem, kmaj(qa, kk), make_sdesc(aHb + kk * 2048, kLinChunk * 128, 1024), id_qh,
                   kk > 0);
          mma_commit(qh_full);
        }
        // state update once the row warps have scaled K by w (after S read it) and the state
        // warps have scaled H by this chunk's g
        mbar_wait(pk_ready, n & 1);
        // Q (read by S and Q Hb, already issued) and the scan arrays: the row warps are past P
        // and the state warps have scaled H by this chunk's g (read from this stage's sL)
        if (n > 0) mbar_wait(h_scaled, (n - 1) & 1);
        mma_commit(&empty[s]);
        mbar_wait(&vfull[s], (n / kSt) & 1);
        AF_LT(3, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem + kColH, make_sdesc(ka + kk * 2048, kLinChunk * 128, 1024),
                 make_sdesc(va + kk * 2048, kLinChunk * 128, 1024), id_h, (n > 0 || kk > 0));
        mma_commit(h_full);
        mma_commit(&kempty[s]);  // Kw: last read by the state update
        if (n > 0) {
          mbar_wait(o_scaled, (n - 1) & 1);
          tc_fence_after();
        }
        AF_LT(2, n);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(o_tmem, tmem + kColS + split_col_lin(kk),
                 make_sdesc(va + kk * 2048, kLinChunk * 128, 1024), id_oi, (n > 0 || kk > 0));
        mma_commit(&oi_full[ob]);
        mma_commit(&vempty[s]);  // V: last read by P V
      }
    }
  } else if (warp >= 12) {
    // ───────────── output warps: O of chunk n -> bf16 rows (+ dot) ─────────────
    const int wq = warp - 12;
    const int r = wq * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    for (int n = 0; n < nchunks; ++n) {
      const int c = chunk_of(n);
      const int t = c * kLinChunk + r;
      const uint32_t ob = n & 1;
      const bool live = t < p.seq;
      const float rs = (p.o_rowscale.ptr != nullptr && live) ? p.o_rowscale.at(b, h, t) : 1.0f;
      mbar_wait_sleep(&oi_full[ob], (n >> 1) & 1);
      if (warp == 12 && lane_id() == 0) AF_LT(9, n);
      tc_fence_after();
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o) + b * p.o_sb + h * p.o_sh +
                            static_cast<int64_t>(live ? t : 0) * p.o_ss;
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        uint32_t oi[32];
        tmem_ld32(tmem + lane_base + kColO + ob * 128 + q * 32, oi);
        tmem_ld_wait();
        if (q == 3) {  // every column read: release the O buffer
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&o_empty[ob]);
        }
        float ov[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) ov[e] = p.out_scale * __uint_as_float(oi[e]);
        if (live) {
          uint4* d4 = reinterpret_cast<uint4*>(orow + q * 32);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            d4[v] = make_uint4(pack_bf16(rs * ov[v * 8 + 0], rs * ov[v * 8 + 1]),
                               pack_bf16(rs * ov[v * 8 + 2], rs * ov[v * 8 + 3]),
                               pack_bf16(rs * ov[v * 8 + 4], rs * ov[v * 8 + 5]),
                               pack_bf16(rs * ov[v * 8 + 6], rs * ov[v * 8 + 7]));
          if (p.dot_x != nullptr) {
            const uint4* x4 = reinterpret_cast<const uint4*>(
                reinterpret_cast<const __nv_bfloat16*>(p.dot_x) + b * p.x_sb + h * p.x_sh +
                static_cast<int64_t>(t) * p.x_ss + q * 32);
            float dotacc = 0.0f;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const uint4 xv = x4[v];
              const uint32_t* xe = reinterpret_cast<const uint32_t*>(&xv);
#pragma unroll
              for (int q2 = 0; q2 < 4; ++q2)
                dotacc += bf16_lo_(xe[q2]) * ov[v * 8 + 2 * q2] +
                          bf16_hi_(xe[q2]) * ov[v * 8 + 2 * q2 + 1];
            }
            const int64_t rows = static_cast<int64_t>(p.batch) * p.heads * p.seq;
            const int64_t at = q * rows + (static_cast<int64_t>(b) * p.heads + h) * p.seq + t;
            p.dot[at] = dotacc;
            if (p.dot2_x != nullptr) {
              const uint4* y4 = reinterpret_cast<const uint4*>(
                  reinterpret_cast<const __nv_bfloat16*>(p.dot2_x) + b * p.x_sb + h * p.x_sh +
                  static_cast<int64_t>(t) * p.x_ss + q * 32);
              float acc2 = 0.0f;
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                const uint4 yv = y4[v];
                const uint32_t* ye = reinterpret_cast<const uint32_t*>(&yv);
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2)
                  acc2 += bf16_lo_(ye[q2]) * ov[v * 8 + 2 * q2] +
                          bf16_hi_(ye[q2]) * ov[v * 8 + 2 * q2 + 1];
              }
              p.dot2[at] = acc2;
            }
          }
        }
      }
      if (warp == 12 && lane_id() == 0) AF_LT(10, n);
    }
  } else if (warp >= 8) {
    // ───────────── state warps: TMEM lane = d_k row of H ─────────────
    const int wq = warp - 8;
    const int dk = wq * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    for (int n = 0; n < nchunks; ++n) {
      // H after chunk n (its update also ends Q Hb of chunk n on the in-order pipe, so Hb may be
      // overwritten): Hb = bf16(H) for chunk n+1's Q Hb, H *= g of chunk n+1
      mbar_wait_sleep(h_full, n & 1);
      if (warp == 8 && lane_id() == 0) AF_LT(16, n);
      tc_fence_after();
      const bool more = n + 1 < nchunks;
      float g = 1.0f;
      if (more) {
        const int s1 = (n + 1) % kSt;
        mbar_wait(&full[s1], ((n + 1) / kSt) & 1);  // chunk n+1's scan arrays
        g = exp2f(sL[s1 * kLinChunk + kLinChunk - 1]);
      }
      const bool last_fwd = !kReverse && !more && p.final_state != nullptr;
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        uint32_t hr[32];
        tmem_ld32(tmem + lane_base + kColH + q * 32, hr);
        tmem_ld_wait();
        if (more) {
          // bf16 copy: row dk of the [d_k][d_v] MN-major B tile (two 64-column SW128 boxes)
          uint8_t* box = sHb + (q / 2) * (kLinChunk * 128);
#pragma unroll
          for (int gq = 0; gq < 4; ++gq)
            *swz_row(box, dk, (q % 2) * 4 + gq) = make_uint4(
                pack_bf16(__uint_as_float(hr[gq * 8 + 0]), __uint_as_float(hr[gq * 8 + 1])),
                pack_bf16(__uint_as_float(hr[gq * 8 + 2]), __uint_as_float(hr[gq * 8 + 3])),
                pack_bf16(__uint_as_float(hr[gq * 8 + 4]), __uint_as_float(hr[gq * 8 + 5])),
                pack_bf16(__uint_as_float(hr[gq * 8 + 6]), __uint_as_float(hr[gq * 8 + 7])));
          uint32_t hs[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) hs[e] = __float_as_uint(__uint_as_float(hr[e]) * g);
          tmem_st32(tmem + lane_base + kColH + q * 32, hs);
        }
        if (last_fwd) {  // the state after the last token (run_step_recurrent's h_S)
          float4* dst = reinterpret_cast<float4*>(
              p.final_state + ((static_cast<int64_t>(b) * p.heads + h) * p.dqk + dk) * p.dv +
              q * 32);
#pragma unroll
          for (int v4 = 0; v4 < 8; ++v4)
            dst[v4] = make_float4(__uint_as_float(hr[v4 * 4]), __uint_as_float(hr[v4 * 4 + 1]),
                                  __uint_as_float(hr[v4 * 4 + 2]), __uint_as_float(hr[v4 * 4 + 3]));
        }
      }
      if (more) {
        fence_proxy_async_smem();
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) {
          mbar_arrive(hb_ready);
          mbar_arrive(h_scaled);
        }
        if (warp == 8 && lane_id() == 0) AF_LT(17, n);
      }
    }
  } else {
    // ───────────── chunk-row warps: two per TMEM lane quarter ─────────────
    const int wq = warp % 4;
    const int half = warp / 4;  // key columns [64 half, +64) of P; O / K columns likewise
    const int r = wq * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    for (int n = 0; n < nchunks; ++n) {
      const int s = n % kSt;
      const uint32_t ob = n & 1;
      mbar_wait(&full[s], (n / kSt) & 1);  // this chunk's scan arrays
      if (threadIdx.x == 0) AF_LT(14, n);
      const float* l = sL + s * kLinChunk;
      const float* u = sU + s * kLinChunk;
      const bool gated = p.ucum != nullptr;
      const float l_r = l[r];
      const float l_last = l[kLinChunk - 1];
      const float cp = kReverse ? exp2f(l_last - l_r) : exp2f(l_r);
      const float g_r = gated ? u[r] : 1.0f;
      const float wgt = g_r * (kReverse ? exp2f(l_r) : exp2f(l_last - l_r));
      // Separable decay: 2^(l_r - l_u) = 2^(l_r - base) 2^(base - l_u) (reverse: the mirror), so
      // P = S a_r b_u with one exponential per row and per column instead of one per element —
      // whenever every l of the chunk is within 2^100 of base (else the per-element form)
      const float base = l[0];
      {
        float dev = fabsf(l_r - base);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dev = fmaxf(dev, __shfl_xor_sync(0xffffffffu, dev, o));
        if (half == 0 && lane_id() == 0) sDev[wq] = dev;
      }
      constexpr uint32_t kRowBar = 1;  // the 8 row warps
      named_bar_sync(kRowBar, 256);
      const bool fac = fmaxf(fmaxf(sDev[0], sDev[1]), fmaxf(sDev[2], sDev[3])) <= 100.0f;
      float a_r = 0.0f;
      if (fac) {
        a_r = kReverse ? ex2(base - l_r) : ex2(l_r - base);
        if (half == 0) sB[r] = (kReverse ? ex2(l_r - base) : ex2(base - l_r)) * g_r;
      }
      // (also orders every warp's sDev read before the next chunk's sDev writes, and the next
      // chunk's sB writes after this chunk's P — a warp reaches them only past this barrier)
      named_bar_sync(kRowBar, 256);
      // (a) P = S o D over this half's 64 key columns
      mbar_wait(s_full, n & 1);
      if (threadIdx.x == 0) AF_LT(7, n);
      tc_fence_after();
      {
        uint32_t pk[32];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int u0 = half * 64 + cc * 32;
          const int r0w = wq * 32;
          const bool none = kReverse ? (u0 + 31 < r0w) : (u0 > r0w + 31);   // all masked
          const bool all = kReverse ? (u0 >= r0w + 31) : (u0 + 31 <= r0w);  // none masked
          if (none) {
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[cc * 16 + e] = 0u;
            continue;
          }
          uint32_t sr[32];
          tmem_ld32(tmem + lane_base + kColS + u0, sr);
          tmem_ld_wait();
          if (fac) {
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              const int uu0 = u0 + e;
              const float4 b4 = *reinterpret_cast<const float4*>(sB + uu0);
              const float bu[4] = {b4.x, b4.y, b4.z, b4.w};
              float pv[4];
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                const bool keep = all || (kReverse ? (uu0 + x >= r) : (uu0 + x <= r));
                pv[x] = keep ? (__uint_as_float(sr[e + x]) * a_r) * bu[x] : 0.0f;
              }
              pk[cc * 16 + e / 2] = pack_bf16(pv[0], pv[1]);
              pk[cc * 16 + e / 2 + 1] = pack_bf16(pv[2], pv[3]);
            }
            continue;
          }
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const int uu0 = u0 + e;
            const float4 l4 = *reinterpret_cast<const float4*>(l + uu0);
            const float4 g4 = gated ? *reinterpret_cast<const float4*>(u + uu0)
                                    : make_float4(1.0f, 1.0f, 1.0f, 1.0f);
            const float lu[4] = {l4.x, l4.y, l4.z, l4.w};
            const float gu[4] = {g4.x, g4.y, g4.z, g4.w};
            float pv[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const bool keep = all || (kReverse ? (uu0 + x >= r) : (uu0 + x <= r));
              const float d = ex2(kReverse ? lu[x] - l_r : l_r - lu[x]) * gu[x];
              pv[x] = keep ? __uint_as_float(sr[e + x]) * d : 0.0f;
            }
            pk[cc * 16 + e / 2] = pack_bf16(pv[0], pv[1]);
            pk[cc * 16 + e / 2 + 1] = pack_bf16(pv[2], pv[3]);
          }
        }
        tmem_st32(tmem + lane_base + kColS + half * 64, pk);  // packed: see split_col_lin
      }
      // (b) Kw = diag(w) K in place, this row's half of the d_k columns (S has read K)
      {
        uint8_t* box = sK + s * L::kTile + half * (kLinChunk * 128);
#pragma unroll
        for (int gq = 0; gq < 8; ++gq) {
          uint4 kv = *swz_row(box, r, gq);
          uint32_t* e = reinterpret_cast<uint32_t*>(&kv);
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2)
            e[q2] = pack_bf16(bf16_lo_(e[q2]) * wgt, bf16_hi_(e[q2]) * wgt);
          *swz_row(box, r, gq) = kv;
        }
      }
      fence_proxy_async_smem();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(pk_ready);
      if (threadIdx.x == 0) AF_LT(8, n);
      // (c) O = Q H_in of this chunk scaled by cp (rows of this half's 64 O columns)
      if (n > 0) {
        mbar_wait(qh_full, (n - 1) & 1);
        if (threadIdx.x == 0) AF_LT(11, n);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const uint32_t col = tmem + lane_base + kColO + ob * 128 + half * 64 + cc * 32;
          uint32_t orr[32];
          tmem_ld32(col, orr);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) orr[e] = __float_as_uint(__uint_as_float(orr[e]) * cp);
          tmem_st32(col, orr);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(o_scaled);
        if (threadIdx.x == 0) AF_LT(12, n);
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

}  // namespace af
