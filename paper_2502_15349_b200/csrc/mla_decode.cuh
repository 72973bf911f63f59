// K3d — MLA decode with the QK^T contraction split across a CTA pair (thread-block cluster of 2).
//
// The 128 x 512 fp32 O accumulator of one token's 128 heads fills TMEM, so each CTA of the pair
// owns one 256-wide value half (as in mla_fwd_kernel<true>).  Instead of both CTAs recomputing
// the full S = Q K^T (576-deep), CTA h contracts only its 288 latent columns:
//   S_h = Q[:, 288h : 288h+288] K[:, 288h : 288h+288]^T        (18 TS k-steps, Q wholly in TMEM)
// and the two partials are exchanged through distributed shared memory: every softmax thread
// stores its row's 32 partial scores into the peer's exchange slot with st.async, whose bytes
// complete the transaction count of the peer's x_full barrier, and adds the peer's partial from
// its own slot once its x_full phase completes.  Both CTAs then hold bit-identical S (fp32 addition commutes) and run the
// same online softmax; each accumulates P V over its value half.  Each CTA streams only the five
// 64-column latent boxes it reads ([0,320) or [256,576)), so the ring holds 6 stages of 32 keys.
//
// TMEM (512 columns): S double buffer [0,64) (P packed in place) | Q[:, 256:288] of this CTA's
// half [64,80) | O half [128,384) | Q[:, 0:256] of the half [384,512).
// Warps: 0-3 softmax rows (one head per thread), 4 TMA, 5 MMA.
#pragma once
#include <cuda.h>

#include "mla.cuh"

namespace af {

constexpr int kDecN = 32;      // keys per tile
constexpr int kDecSt = 6;      // latent ring stages
constexpr int kDecQK = 288;    // contraction columns per CTA of the pair
constexpr int kDecBoxes = 5;   // 64-column latent boxes per CTA

struct MlaDecSmem {
  static constexpr int kKBox = kDecN * 128;           // [32 keys][64 cols] bf16
  static constexpr int kKBytes = kDecBoxes * kKBox;   // 20 KB per stage
  static constexpr int kKOff = 0;
  static constexpr int kXOff = kKOff + kDecSt * kKBytes;        // exchange [2][128 rows][32] fp32
  static constexpr int kBarOff = kXOff + 2 * 128 * kDecN * 4;
  // k_full[St], k_empty[St], s_full[2], x_full[2], x_empty[2], q_ready, p_ready, o_done
  static constexpr int kNumBars = 2 * kDecSt + 9;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
};

AF_DEVICE uint32_t cluster_map(uint32_t local_smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem_addr), "r"(rank));
  return r;
}
// 16-byte store into a peer CTA's shared memory that counts its bytes on the peer's mbarrier
// (complete_tx): the receiver's plain phase wait then also covers the data's visibility.
AF_DEVICE void st_async_v4(uint32_t addr, uint32_t remote_bar, float a, float b, float c, float d) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::
          "r"(addr),
      "f"(a), "f"(b), "f"(c), "f"(d), "r"(remote_bar)
      : "memory");
}
AF_DEVICE void mbar_arrive_cluster(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar)
               : "memory");
}
AF_DEVICE void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
AF_DEVICE void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    mla_decode_pair_kernel(const __grid_constant__ CUtensorMap tm_kv, const MlaParams p) {
  using L = MlaDecSmem;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + L::kKOff;
  float* sX = reinterpret_cast<float*>(smem + L::kXOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* k_full = bars;
  uint64_t* k_empty = bars + kDecSt;
  uint64_t* s_full = bars + 2 * kDecSt;  // [2]
  uint64_t* x_full = s_full + 2;         // [2]: the peer's partial landed in my slot
  uint64_t* x_empty = x_full + 2;        // [2]: the peer consumed the slot I wrote
  uint64_t* q_ready = x_empty + 2;
  uint64_t* p_ready = q_ready + 1;
  uint64_t* o_done = p_ready + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);

  const int warp = static_cast<int>(warp_id());
  const uint32_t half = blockIdx.x & 1;  // == cluster rank: value half and contraction half
  const uint32_t peer = half ^ 1;
  const int rest = blockIdx.x >> 1;
  const int split = rest % p.splits;
  const int b = rest / p.splits;
  const int kv_lo = split * p.split_len;
  const int kv_hi = min(p.seq_k, kv_lo + p.split_len);
  const int nk = kv_hi > kv_lo ? (kv_hi - kv_lo + kDecN - 1) / kDecN : 0;

  if (warp == 4 && lane_id() == 0) {
    for (int s = 0; s < kDecSt; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&x_full[s], 1);  // local expect_tx arrive + the peer's st.async bytes
      mbar_init(&x_empty[s], 128);
    }
    mbar_init(q_ready, 4);
    mbar_init(p_ready, 4);
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync_all();  // the peer's barriers are initialised before any remote arrive
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kColO = 128, kColQ = 384;
  // TMEM column of this CTA's packed Q chunk c (64 contraction columns; chunk 4 is 32 wide)
  auto q_tcol = [](int c) -> uint32_t { return c < 4 ? kColQ + c * 32 : 64u; };

  if (warp == 4) {
    if (elect_one() && nk > 0) {
      for (int n = 0; n < nk; ++n) {
        const int s = n % kDecSt;
        mbar_wait(&k_empty[s], ((n / kDecSt) & 1) ^ 1);
        mbar_expect_tx(&k_full[s], L::kKBytes);
        const int j0 = kv_lo + n * kDecN;
        for (int c = 0; c < kDecBoxes; ++c)
          tma_load_4d_hint(sK + s * L::kKBytes + c * L::kKBox, &tm_kv, &k_full[s],
                           (static_cast<int>(half) * 4 + c) * 64, j0, b, 0, kEvictLast);
      }
    }
  } else if (warp == 5) {
    if (elect_one() && nk > 0) {
      constexpr uint32_t id_s = make_idesc_bf16(128, kDecN, false, false);    // S_h = Q_h K_h^T
      constexpr uint32_t id_o = make_idesc_bf16(128, kMlaHalf, false, true);  // O_h += P V_h
      const uint32_t aK = smem_u32(sK);
      // local latent column of contraction k-step kk: half 1's boxes start at column 256 and
      // its contraction at 288
      const int dl0 = half ? 32 : 0;
      auto issue_s = [&](int n) {
        const int s = n & 1;
        const int st = n % kDecSt;
        mbar_wait(&k_full[st], (n / kDecSt) & 1);
        tc_fence_after();
        const uint32_t kb = aK + st * L::kKBytes;
#pragma unroll
        for (int kk = 0; kk < kDecQK / 16; ++kk) {
          const int dl = dl0 + kk * 16;
          mma_ts(tmem + s * kDecN, tmem + q_tcol(kk / 4) + (kk % 4) * 8,
                 make_sdesc(kb + (dl / 64) * L::kKBox + ((dl % 64) / 16) * 32, 0, 1024), id_s,
                 kk > 0);
        }
        mma_commit(&s_full[s]);
      };
      mbar_wait(q_ready, 0);
      tc_fence_after();
      issue_s(0);
      for (int n = 0; n < nk; ++n) {
        const int s = n & 1;
        const int st = n % kDecSt;
        if (n + 1 < nk) issue_s(n + 1);
        mbar_wait(p_ready, n & 1);
        tc_fence_after();
        // V half = local latent columns [0, 256) of either CTA (boxes 0..3), MN-major
        const uint32_t vbase = aK + st * L::kKBytes;
#pragma unroll
        for (int kk = 0; kk < kDecN / 16; ++kk)
          mma_ts(tmem + kColO, tmem + s * kDecN + kk * 8,
                 make_sdesc(vbase + kk * 2048, L::kKBox, 1024), id_o, (n > 0 || kk > 0));
        mma_commit(o_done);
        mma_commit(&k_empty[st]);
      }
    }
  } else {
    // ───────────── softmax rows: one head per thread ─────────────
    const int row = warp * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    {  // this CTA's 288 contraction columns of Q -> TMEM (packed bf16 pairs, A-operand layout)
      const bool live = row < p.heads;
      const __nv_bfloat16* qrow =
          p.q + b * p.q_sb + static_cast<int64_t>(live ? row : 0) * p.q_ss + half * kDecQK;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t w[32];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint4 x = live ? *reinterpret_cast<const uint4*>(qrow + c * 64 + v * 8)
                               : make_uint4(0u, 0u, 0u, 0u);
          w[v * 4 + 0] = x.x;
          w[v * 4 + 1] = x.y;
          w[v * 4 + 2] = x.z;
          w[v * 4 + 3] = x.w;
        }
        tmem_st32(tmem + lane_base + q_tcol(c), w);
      }
      uint32_t w[16];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint4 x = live ? *reinterpret_cast<const uint4*>(qrow + 256 + v * 8)
                             : make_uint4(0u, 0u, 0u, 0u);
        w[v * 4 + 0] = x.x;
        w[v * 4 + 1] = x.y;
        w[v * 4 + 2] = x.z;
        w[v * 4 + 3] = x.w;
      }
      tmem_st16(tmem + lane_base + q_tcol(4), w);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(q_ready);
    }
    // exchange slot of this row: [slot][row][32] fp32, 16-byte granules swizzled by row
    auto xaddr = [&](int slot, int g) -> float* {
      return sX + (slot * 128 + row) * kDecN + ((g ^ (row & 7)) * 4);
    };
    const uint32_t peer_x_full0 = cluster_map(smem_u32(&x_full[0]), peer);
    const uint32_t peer_x_empty0 = cluster_map(smem_u32(&x_empty[0]), peer);
    float m_run = -INFINITY, l_run = 0.0f;
    for (int n = 0; n < nk; ++n) {
      const int s = n & 1;
      const int j0 = kv_lo + n * kDecN;
      mbar_wait(&s_full[s], (n >> 1) & 1);
      tc_fence_after();
      uint32_t sr[kDecN];
      tmem_ld32(tmem + lane_base + s * kDecN, sr);
      tmem_ld_wait();
      // this tile's incoming bytes on my slot s: 128 rows x 32 fp32
      if (row == 0) mbar_expect_tx(&x_full[s], 128 * kDecN * 4);
      // hand this CTA's partial to the peer (its slot s may be reused once the peer read it)
      if (n >= 2) mbar_wait_cluster(&x_empty[s], ((n >> 1) - 1) & 1);
      const uint32_t rbar = peer_x_full0 + s * 8;
#pragma unroll
      for (int g = 0; g < kDecN / 4; ++g)
        st_async_v4(cluster_map(smem_u32(xaddr(s, g)), peer), rbar, __uint_as_float(sr[g * 4]),
                    __uint_as_float(sr[g * 4 + 1]), __uint_as_float(sr[g * 4 + 2]),
                    __uint_as_float(sr[g * 4 + 3]));
      // the peer's partial: S = S_own + S_peer (the same sum on both CTAs)
      mbar_wait(&x_full[s], (n >> 1) & 1);
      float x[kDecN];
#pragma unroll
      for (int g = 0; g < kDecN / 4; ++g) {
        const float4 o4 = *reinterpret_cast<const float4*>(xaddr(s, g));
        x[g * 4 + 0] = __uint_as_float(sr[g * 4 + 0]) + o4.x;
        x[g * 4 + 1] = __uint_as_float(sr[g * 4 + 1]) + o4.y;
        x[g * 4 + 2] = __uint_as_float(sr[g * 4 + 2]) + o4.z;
        x[g * 4 + 3] = __uint_as_float(sr[g * 4 + 3]) + o4.w;
      }
      mbar_arrive_cluster(peer_x_empty0 + s * 8);
      float bmax = -INFINITY;
      const bool full = j0 + kDecN <= kv_hi;
#pragma unroll
      for (int e = 0; e < kDecN; ++e) {
        const bool keep = full || (j0 + e < kv_hi);
        x[e] = keep ? x[e] * p.scale_log2 : -INFINITY;
        bmax = fmaxf(bmax, x[e]);
      }
      const float m_new = fmaxf(m_run, bmax);
      const bool need = (m_new - m_run) > 8.0f;
      float factor = 1.0f;
      if (need) {
        factor = (m_run == -INFINITY) ? 0.0f : ex2(m_run - m_new);
        m_run = m_new;
      }
      const float m_use = (m_run == -INFINITY) ? 0.0f : m_run;
      uint32_t pk[kDecN / 2];
      float lsum = 0.0f;
#pragma unroll
      for (int e = 0; e < kDecN; e += 2) {
        const float e0 = ex2(x[e] - m_use), e1 = ex2(x[e + 1] - m_use);
        lsum += e0 + e1;
        pk[e / 2] = pack_bf16(e0, e1);
      }
      l_run = l_run * factor + lsum;
      tmem_st16(tmem + lane_base + s * kDecN, pk);
      tmem_st_wait();
      if (n > 0 && __any_sync(0xffffffffu, need)) {
        mbar_wait(o_done, (n - 1) & 1);
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
      if (lane_id() == 0) mbar_arrive(p_ready);
    }
    // ───────────── epilogue: this half's normalised partial O and (half 0) the LSE ─────────────
    if (nk > 0) {
      mbar_wait(o_done, (nk - 1) & 1);
      tc_fence_after();
    }
    const float inv = (l_run == 0.0f) ? 0.0f : 1.0f / l_run;
    const float lse = (l_run == 0.0f) ? -INFINITY : (m_run * kLn2 + logf(l_run));
    float* dst = p.part_o + ((static_cast<int64_t>(b) * p.splits + split) * p.heads + row) * kMlaDv +
                 half * kMlaHalf;
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
      if (row < p.heads) {
        float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          d4[v] = make_float4(__uint_as_float(orr[v * 4]) * inv, __uint_as_float(orr[v * 4 + 1]) * inv,
                              __uint_as_float(orr[v * 4 + 2]) * inv,
                              __uint_as_float(orr[v * 4 + 3]) * inv);
      }
    }
    if (half == 0 && row < p.heads)
      p.part_lse[(static_cast<int64_t>(b) * p.splits + split) * p.heads + row] = lse;
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while its peer may still write its slots / barriers
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace af
