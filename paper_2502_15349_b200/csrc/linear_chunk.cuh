// K4 — linear (recurrent) template on sm_100a: chunked linear attention with a carried state.
//
// Computes, per (b, h) and per 64-wide block of the value dimension,
//   forward : o_t = s_out * sum_{u<=t} e^{L_t - L_u} (q_t . k_u) v_u
//   reverse : o_t = s_out * sum_{u>=t} e^{L_u - L_t} (q_t . k_u) v_u
// with L the inclusive cumsum of log a_t — the recurrence h_t = a_t h_{t-1} + k_t^T v_t,
// o_t = q_t h_t of attnforge `engine.run_step_recurrent` (engine.py:525-551), evaluated the way
// `engine.run_chunk_recurrent` does (engine.py:554-616): per chunk of C = 128 tokens,
//   O_c   = ((Q K^T) o D) V + (Q o cp) H_in        D[i,u] = e^{l_i - l_u} [u <= i]
//   H_out = g H_in + (K o w)^T V                    cp_i = e^{l_i}, w_u = e^{l_{C-1} - l_u}, g = e^{l_{C-1}}
// (l = in-chunk inclusive cumsum; the reverse direction swaps the roles, see below).  The
// backward of the template is three more runs of this kernel (restated):
//   dQm = LA_fwd(q=dO, k=V, v=Km),  dKm = LA_rev(q=V, k=dO, v=Qm),  dV = LA_rev(q=Km, k=Qm, v=dO),
//   d log a_t = sum_{s>=t} (Qm_s . dQm_s - Km_s . dKm_s)
// — the optional `dot` output accumulates X_t . o_t (fp32) for that last line.
//
// One CTA owns one (b, h, value block) and walks the chunks in order (reverse: last to first),
// carrying the [DK x 64] fp32 state in TMEM.  Warps 0-7: two per chunk row (= TMEM lane), each
// owning one half of the columns (scan of log a, decay weights, P = S o D, state rescale, bf16
// state copy); warps 8-11: output epilogue of the previous chunk (OI / QH double-buffered);
// warp 12: TMA producer; warp 13: TMEM allocator + MMA issuer.
// TMEM: S [0,128) (packed P) | OI [128,192) | QH x2 [192,320) | H [320, 320+64*DK/128)
// MMAs (all M=128): S = Q K^T (SS), QH = Q Hb (SS, Hb = bf16 state copy in smem), OI = P V (TS),
// H += K^T Vw (SS, K^T read MN-major straight from the K tile, Vw = diag(w) V).
#pragma once
#include <cuda.h>
#include "params.h"
#include "sm100.cuh"

namespace af {

#ifdef AF_TRACE
// Developer timeline of CTA 0: g_lin_trace[event][chunk] = clock64().
__device__ long long g_lin_trace[24][128];
#define AF_LT(ev, n)                                                                  \
  do {                                                                                \
    if (blockIdx.x == 0 && (n) < 128) g_lin_trace[ev][n] = clock64();                 \
  } while (0)
#else
#define AF_LT(ev, n) \
  do {               \
  } while (0)
#endif

constexpr int kLinChunk = 128;
constexpr int kRawRing = 4;  // chunks of raw per-step factors in flight (producer warp)
// Waits of warps that idle for long stretches (row warps between chunks, output warps, loaders):
// with a back-off they stop taking issue slots from the scan warp on their SMSP.
#ifndef AF_LIN_IDLE_SLEEP
#define AF_LIN_IDLE_SLEEP 1
#endif
#if AF_LIN_IDLE_SLEEP
#define LIN_IDLE_WAIT(bar, par) mbar_wait_sleep(bar, par)
#else
#define LIN_IDLE_WAIT(bar, par) mbar_wait(bar, par)
#endif
constexpr int kLinVB = 64;  // value columns per CTA

// Per-step fp32 tensor with element strides [b, h, s] (0 = broadcast axis).
struct StepTensor {
  const float* ptr;
  int64_t sb, sh, ss;
  AF_DEVICE float at(int b, int h, int t) const { return ptr[b * sb + h * sh + t * ss]; }
};

struct LinearParams {
  int batch, heads, seq, dqk, dv;
  float out_scale;
  // log a_t = log_const + sum_f log(fac[f][b, h, t])
  float log_const;
  int nfac;
  StepTensor fac[2];
  StepTensor u_scale;    // per-token scale of the key/value side (k_mod = k * gate); ptr may be null
  StepTensor o_rowscale; // per-token scale of the output rows (not of `dot`); ptr may be null
  void* o;              // bf16 output with element strides
  int64_t o_sb, o_sh, o_ss;
  const void* dot_x;    // optional bf16 X with element strides: dot[t] += X_t . o_t
  int64_t x_sb, x_sh, x_ss;
  float* final_state;   // optional fp32 [B, H, dqk, dv]: the state after the last token (forward)
  const void* dot2_x;   // optional second X (same strides as dot_x): dot2[t] = X2_t . o_t — the
  float* dot2;          // backward's raw-key dot of the gate gradient (same slot layout as dot)
  float* dot;           // [dv/32 slots][B, H, S] fp32: one partial per 32-column slot, summed
                        // in slot order by linear_step_grads_kernel (deterministic)
  // the decay scan of linear_decay_scan_kernel, [B*H][nchunks][128] (padded tail: a = 1, u = 1)
  const float* lcum;    // in-chunk inclusive cumsum of log2 a
  const float* ucum;    // key/value-side scale u (k_mod gate); null when absent
  const int* cflag;     // [B*H][nchunks]: 1 when every |L| of the chunk is <= 100
};

template <int DK>
struct LinSmem {
  static constexpr int kStages = DK == 128 ? 2 : 1;   // Q/K ring depth (smem bound at DK=256)
  static constexpr int kVStages = DK == 128 ? 3 : 2;  // V ring: released later (after O I), deeper
  static constexpr int kQBytes = kLinChunk * DK * 2;
  static constexpr int kVBytes = kLinChunk * kLinVB * 2;
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + kStages * kQBytes;
  static constexpr int kVOff = kKOff + kStages * kQBytes;
  static constexpr int kVwOff = kVOff + kVStages * kVBytes;
  static constexpr int kHbOff = kVwOff + kVBytes;
  // [2 chunks in flight][128]: in-chunk cumsum of log2 a, key/value-side scale, and the column
  // factor e^{-+L_u} u_u of the factorised decay — scanned by the producer warp one chunk ahead
  static constexpr int kLOff = kHbOff + DK * kLinVB * 2;
  static constexpr int kUOff = kLOff + 2 * kLinChunk * 4;
  static constexpr int kEcOff = kUOff + 2 * kLinChunk * 4;
  static constexpr int kRawOff = kEcOff + 2 * kLinChunk * 4;  // [kRawRing][3][128] raw factors
  static constexpr int kCpOff = kRawOff + kRawRing * 3 * kLinChunk * 4;  // [2][128] output decay
  static constexpr int kFlagOff = kCpOff + 2 * kLinChunk * 4;
  // ring: full[S], empty[S]; s_full qh_full oi_full[2] h_full scan_ready[2] (raw factors of the
  // chunk landed; 1 arrival) | p_ready vw_ready h_scaled hb_ready scan_free[2] (raw factors read;
  // 8 row warps) | oi_empty[2] cp_ready[2] (4)
  static constexpr int kBarOff = kFlagOff + 32;
  static constexpr int kNumBars = 2 * kStages + 17 + 2 * kVStages;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kTotal = kTmemSlotOff + 16;
};

constexpr float kLog2e_ = 1.4426950408889634f;

// log2 of a per-step decay factor, floored at -200: a factor of exactly 0 (a state reset) gives
// 2^-200 = 0 in fp32 after the cumulative sums instead of -inf - -inf = NaN.  A negative factor
// stays NaN (log-space decays need a >= 0; the host reports it as unsupported).
AF_DEVICE float log2_floor(float v) {
  const float l = __log2f(v);
  return l < -200.0f ? -200.0f : l;
}

// The per-step decay scan, once per call for every chunk in parallel (one warp per (b, h, chunk)):
// L = in-chunk inclusive cumsum of log2 a_t (a_t = e^{log_const} prod_f fac_f[t]), the key/value
// scale u_t, and a per-chunk flag for the factorised-decay path (every |L| <= 100).  Traced inside
// the chunk kernel this serial LDS / MUFU / SHFL chain held a whole chunk period (~1.8k clk of a
// single latency-bound warp); here it runs ahead of every template pass that shares the decay
// (the forward, and all three passes of the backward).
__global__ void linear_decay_scan_kernel(const LinearParams p, float* __restrict__ lcum,
                                         float* __restrict__ ucum, int* __restrict__ cflag) {
  const int lane = static_cast<int>(threadIdx.x & 31);
  const int nchunks = (p.seq + kLinChunk - 1) / kLinChunk;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  if (gw >= static_cast<int64_t>(p.batch) * p.heads * nchunks) return;
  const int c = static_cast<int>(gw % nchunks);
  const int bh = static_cast<int>(gw / nchunks);
  const int b = bh / p.heads, h = bh % p.heads;
  float x[4], us[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int t = c * kLinChunk + lane * 4 + j;
    x[j] = 0.0f;
    us[j] = 1.0f;
    if (t < p.seq) {
      x[j] = p.log_const * kLog2e_;
#pragma unroll
      for (int f = 0; f < 2; ++f)
        if (f < p.nfac) x[j] += log2_floor(p.fac[f].at(b, h, t));
      if (p.u_scale.ptr != nullptr) us[j] = p.u_scale.at(b, h, t);
    }
  }
  x[1] += x[0];
  x[2] += x[1];
  x[3] += x[2];
  float tot = x[3];
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, tot, off);
    if (lane >= off) tot += y;
  }
  const float excl = tot - x[3];
  float amax = fmaxf(fabsf(excl + x[0]), fabsf(excl + x[3]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  reinterpret_cast<float4*>(lcum + gw * kLinChunk)[lane] =
      make_float4(excl + x[0], excl + x[1], excl + x[2], excl + x[3]);
  if (ucum != nullptr)
    reinterpret_cast<float4*>(ucum + gw * kLinChunk)[lane] = make_float4(us[0], us[1], us[2], us[3]);
  if (lane == 0) cflag[gw] = amax <= 100.0f ? 1 : 0;
}

// packed (bf16x2) TMEM column of the k-th 16-key slice of P (key halves [0,64) -> [0,32),
// [64,128) -> [64,96): each row-warp half only overwrites S columns it alone has read)
AF_DEVICE uint32_t split_col_lin(int kk) { return kk < 4 ? kk * 8 : 64 + (kk - 4) * 8; }

// 128-byte-row swizzled tile helpers ([rows][64 bf16], 16-byte granule g of row r stored at
// granule g ^ (r % 8) — the layout TMA SWIZZLE_128B produces and UMMA descriptors expect).
AF_DEVICE uint4* swz_row(uint8_t* base, int r, int g) {
  return reinterpret_cast<uint4*>(base + r * 128 + ((g ^ (r & 7)) << 4));
}

// Warp roles: 0-7 chunk-row warps (two per TMEM lane quarter), 8-11 output warps (one per lane
// quarter: O = s_out (OI + cp Q H) of chunk n runs while the row warps already work on chunk n+1;
// OI and QH are double-buffered in TMEM), 12 per-step decay scan, 13 TMEM allocator + MMA issuer,
// 14 TMA loader of Q/K, 15 TMA loader of V.  The loaders run ahead of the scan by the ring depths
// (a single producer issuing the loads behind the scan left V late: ncu's top stall was the row
// warps waiting on vfull; cfg5b fwd 0.473 -> 0.448 ms).
// DK = 256 (single-stage Q/K ring) keeps the loads in warp 12 and runs without warps 14-15.
__host__ __device__ constexpr int lin_threads(int dk) { return dk == 128 ? 512 : 448; }

template <int DK, bool kReverse, bool kFac>
__global__ void __launch_bounds__(lin_threads(DK), 1)
    linear_chunk_kernel(const __grid_constant__ CUtensorMap tm_q,
                        const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const LinearParams p) {
  using L = LinSmem<DK>;
  static_assert(DK == 128 || DK == 256, "DK");
  constexpr int kHalves = DK / 128;
  constexpr int kStages = L::kStages;
  // DK = 128 (two-stage Q/K ring): dedicated loader warps run ahead of the scan; DK = 256 (one
  // stage) keeps the loads behind the scan in warp 12 (measured: the loaders' spinning cost more
  // than the run-ahead gained there)
  constexpr bool kSplitLoad = lin_threads(DK) == 512;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint8_t* sVw = smem + L::kVwOff;
  uint8_t* sHb = smem + L::kHbOff;
  float* sLb = reinterpret_cast<float*>(smem + L::kLOff);  // [2][128]
  float* sUb = reinterpret_cast<float*>(smem + L::kUOff);  // [2][128]
  float* sRaw = reinterpret_cast<float*>(smem + L::kRawOff);
  float* sCp = reinterpret_cast<float*>(smem + L::kCpOff);
  float* sEcb = reinterpret_cast<float*>(smem + L::kEcOff);  // [2][128]
  volatile int* sFac = reinterpret_cast<volatile int*>(smem + L::kFlagOff);  // [2][4 groups]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* full = bars;                 // Q, K, V of one chunk landed (one tx barrier)
  uint64_t* empty = bars + kStages;      // the chunk's Q, K, V may be overwritten
  uint64_t* s_full = bars + 2 * kStages;
  uint64_t* qh_full = s_full + 1;
  uint64_t* oi_full = s_full + 2;        // [2]
  uint64_t* h_full = s_full + 4;
  uint64_t* p_ready = s_full + 5;
  uint64_t* vw_ready = s_full + 6;
  uint64_t* h_scaled = s_full + 7;
  uint64_t* hb_ready = s_full + 8;
  uint64_t* oi_empty = s_full + 9;       // [2]
  uint64_t* cp_ready = s_full + 11;      // [2]
  uint64_t* scan_ready = s_full + 13;    // [2]
  uint64_t* scan_free = s_full + 15;     // [2]
  constexpr int kVSt = L::kVStages;
  uint64_t* vfull = s_full + 17;         // [kVSt]: V of one chunk landed
  uint64_t* vempty = vfull + kVSt;       // [kVSt]: that V may be overwritten
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlotOff);

  const int warp = static_cast<int>(warp_id());
  const int nvb = p.dv / kLinVB;
  const int vb = blockIdx.x % nvb;
  const int bh = blockIdx.x / nvb;
  const int b = bh / p.heads;
  const int h = bh % p.heads;
  const int nchunks = (p.seq + kLinChunk - 1) / kLinChunk;

  if (warp == 12 && lane_id() == 0) {
    for (int i = 0; i < 2 * kStages + 5; ++i) mbar_init(&bars[i], 1);
    for (int i = 2 * kStages + 5; i < 2 * kStages + 9; ++i) mbar_init(&bars[i], 8);
    for (int i = 2 * kStages + 9; i < 2 * kStages + 13; ++i) mbar_init(&bars[i], 4);
    mbar_init(&scan_ready[0], 1);
    mbar_init(&scan_ready[1], 1);
    mbar_init(&scan_free[0], 8);
    mbar_init(&scan_free[1], 8);
    for (int i = 0; i < kVSt; ++i) {
      mbar_init(&vfull[i], 1);
      mbar_init(&vempty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 13) tmem_alloc<512>(tmem_slot);
  if (warp < 8) {  // zero the bf16 state copy: chunk 0 multiplies Q by H_in = 0
    for (int i = threadIdx.x; i < DK * kLinVB * 2 / 16; i += 256)
      reinterpret_cast<uint4*>(sHb)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // S [0,128) | OI x2 [128,256) | QH x2 [256,384) | H [384, 384 + 64*DK/128)
  constexpr uint32_t kColS = 0, kColOI = 128, kColQH = 256, kColH = 384;

  if (warp == 12) {
    // ───────────── producer warp: per-step decay scan (+ the TMA ring at DK = 256) ─────────────
    // Chunk n's raw factors land by cp.async; this warp then scans them — L = in-chunk inclusive
    // cumsum of log2 a, the key/value-side scale u and, when the chunk's |L| stays below 2^100,
    // the column factors e^{-+L_u} u_u of the factorised decay — into the shared [n % 2] arrays,
    // one chunk ahead of the row warps (traced: a scan inside every row warp put ~2.5k clk of
    // dependent LDS / MUFU / SHFL latency on the ~6k-clk chunk period).
    const int lane = static_cast<int>(lane_id());
    const int nraw = p.nfac + (p.u_scale.ptr != nullptr ? 1 : 0);
    // the precomputed scan (linear_decay_scan_kernel) of chunk n lands in ring slot n % kRawRing
    // by cp.async, kRawRing - 1 chunks ahead; this warp turns it into the shared [n % 2] arrays
    // the row warps read (L, u and the column factors of the factorised decay)
    const int bhx = b * p.heads + h;
    auto load_raw = [&](int m) {
      if (m < nchunks) {
        const int cm = kReverse ? nchunks - 1 - m : m;
        const int64_t g = static_cast<int64_t>(bhx) * nchunks + cm;
        float* raw = sRaw + (m % kRawRing) * 3 * kLinChunk;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(raw + lane * 4)),
                     "l"(p.lcum + g * kLinChunk + lane * 4)
                     : "memory");
        if (p.ucum != nullptr)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           smem_u32(raw + kLinChunk + lane * 4)),
                       "l"(p.ucum + g * kLinChunk + lane * 4)
                       : "memory");
        if (lane == 0)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                           smem_u32(raw + 2 * kLinChunk)),
                       "l"(p.cflag + g)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");  // (empty groups keep the count)
    };
    for (int m = 0; m < kRawRing - 1; ++m) load_raw(m);
    for (int n = 0; n < nchunks; ++n) {
      const int c = kReverse ? nchunks - 1 - n : n;
      const int t0 = c * kLinChunk;
      const int pb = n & 1;
      load_raw(n + kRawRing - 1);  // its slot held chunk n-1, already consumed by this warp
      asm volatile("cp.async.wait_group %0;" ::"n"(kRawRing - 1) : "memory");
      __syncwarp();
      if (lane == 0) AF_LT(17, n);
      const float* raw = sRaw + (n % kRawRing) * 3 * kLinChunk;
      {
        const float4 l4 = reinterpret_cast<const float4*>(raw)[lane];
        const float4 u4 = p.ucum != nullptr ? reinterpret_cast<const float4*>(raw + kLinChunk)[lane]
                                            : make_float4(1.0f, 1.0f, 1.0f, 1.0f);
        const float lj4[4] = {l4.x, l4.y, l4.z, l4.w};
        const float us[4] = {u4.x, u4.y, u4.z, u4.w};
        // Factorised decay per 32-key group g (base index b_g: the group's first key, reverse:
        // its last): D[i,u] = 2^{L_i - L_bg} * 2^{L_bg - L_u} (reverse: 2^{L_bg - L_i} *
        // 2^{L_u - L_bg}).  The column factor 2^{+-(L_bg - L_u)} u_u is built here; the row
        // warps multiply by their one row factor per group — an ex2 per element only in groups
        // whose decay spans more than 2^100 (the column factor would leave fp32's range).  Row
        // factors of kept pairs are <= 1, so nothing overflows; underflow only drops terms
        // below 2^-26 of the diagonal's.
        const int gl = lane & ~7;  // first lane of this lane's 32-key group
        const float base = kReverse ? __shfl_sync(0xffffffffu, lj4[3], gl + 7)
                                    : __shfl_sync(0xffffffffu, lj4[0], gl);
        float dmax = 0.0f;
#pragma unroll
        for (int j = 0; j < 4; ++j) dmax = fmaxf(dmax, fabsf(lj4[j] - base));
#pragma unroll
        for (int off = 1; off < 8; off <<= 1)
          dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
        const bool gfac = dmax <= 100.0f;
        if (n >= 2) LIN_IDLE_WAIT(&scan_free[pb], ((n >> 1) - 1) & 1);  // chunk n-2 fully read
        if (lane == 0) AF_LT(16, n);
        float* sL = sLb + pb * kLinChunk;
        float* sU = sUb + pb * kLinChunk;
        float* sEc = sEcb + pb * kLinChunk;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float lj = lj4[j];
          sL[lane * 4 + j] = lj;
          sU[lane * 4 + j] = us[j];
          if (gfac) sEc[lane * 4 + j] = exp2f(kReverse ? lj - base : base - lj) * us[j];
        }
        if (lane == gl) sFac[pb * 4 + (lane >> 3)] = gfac ? 1 : 0;
        __syncwarp();
      }
      if (lane == 0) mbar_arrive(&scan_ready[pb]);
      if (lane == 0) AF_LT(15, n);
      if constexpr (!kSplitLoad) {  // Q, K, V of chunk n behind its scan (single-stage Q/K ring)
        if (elect_one()) {
          const int st = n % kStages;
          mbar_wait(&empty[st], ((n / kStages) & 1) ^ 1);
          mbar_expect_tx(&full[st], 2 * L::kQBytes);
          for (int x = 0; x < DK / 64; ++x) {
            tma_load_4d(sQ + st * L::kQBytes + x * (kLinChunk * 128), &tm_q, &full[st], x * 64,
                        t0, h, b);
            tma_load_4d(sK + st * L::kQBytes + x * (kLinChunk * 128), &tm_k, &full[st], x * 64,
                        t0, h, b);
          }
          const int sv = n % kVSt;
          mbar_wait(&vempty[sv], ((n / kVSt) & 1) ^ 1);
          mbar_expect_tx(&vfull[sv], L::kVBytes);
          tma_load_4d(sV + sv * L::kVBytes, &tm_v, &vfull[sv], vb * kLinVB, t0, h, b);
        }
        __syncwarp();
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else if (warp == 14 || warp == 15) {
    // ───────────── TMA loaders: Q/K ring (warp 14), V ring (warp 15) ─────────────
    if (kSplitLoad && elect_one()) {
      for (int n = 0; n < nchunks; ++n) {
        const int c = kReverse ? nchunks - 1 - n : n;
        const int t0 = c * kLinChunk;
        if (warp == 14) {
          const int st = n % kStages;
          LIN_IDLE_WAIT(&empty[st], ((n / kStages) & 1) ^ 1);
          mbar_expect_tx(&full[st], 2 * L::kQBytes);
          for (int x = 0; x < DK / 64; ++x) {
            tma_load_4d(sQ + st * L::kQBytes + x * (kLinChunk * 128), &tm_q, &full[st], x * 64,
                        t0, h, b);
            tma_load_4d(sK + st * L::kQBytes + x * (kLinChunk * 128), &tm_k, &full[st], x * 64,
                        t0, h, b);
          }
        } else {
          const int sv = n % kVSt;
          LIN_IDLE_WAIT(&vempty[sv], ((n / kVSt) & 1) ^ 1);
          mbar_expect_tx(&vfull[sv], L::kVBytes);
          tma_load_4d(sV + sv * L::kVBytes, &tm_v, &vfull[sv], vb * kLinVB, t0, h, b);
        }
      }
    }
  } else if (warp == 13) {
    // ───────────── MMA issuer:  S | QH | H update | OI ─────────────
    if (elect_one()) {
      constexpr uint32_t id_s = make_idesc_bf16(128, 128, false, false);     // S = Q K^T
      constexpr uint32_t id_qh = make_idesc_bf16(128, kLinVB, false, true);  // QH = Q Hb
      constexpr uint32_t id_oi = make_idesc_bf16(128, kLinVB, false, true);  // OI = P V
      constexpr uint32_t id_h = make_idesc_bf16(128, kLinVB, true, true);    // H += K^T Vw
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV);
      const uint32_t aVw = smem_u32(sVw), aHb = smem_u32(sHb);
      auto kmaj = [](uint32_t base, int kk) {
        return make_sdesc(base + (kk / 4) * (kLinChunk * 128) + (kk % 4) * 32, 0, 1024);
      };
      for (int n = 0; n < nchunks; ++n) {
        const uint32_t ph = n & 1;
        const int st = n % kStages;
        const uint32_t qa = aQ + st * L::kQBytes, ka = aK + st * L::kQBytes;
        const int sv = n % kVSt;
        const uint32_t va = aV + sv * L::kVBytes;
        mbar_wait(&full[st], (n / kStages) & 1);
        AF_LT(0, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DK / 16; ++kk)
          mma_ss(tmem + kColS, kmaj(qa, kk), kmaj(ka, kk), id_s, kk > 0);
        mma_commit(s_full);
        if (n > 0) mbar_wait(hb_ready, (n - 1) & 1);
        if (n >= 2) mbar_wait(&oi_empty[ph], ((n >> 1) - 1) & 1);  // chunk n-2's output read
        AF_LT(1, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DK / 16; ++kk)
          mma_ss(tmem + kColQH + ph * kLinVB, kmaj(qa, kk),
                 make_sdesc(aHb + kk * 2048, 16384, 1024), id_qh, kk > 0);
        mma_commit(qh_full);
        mbar_wait(vw_ready, ph);
        mbar_wait(h_scaled, ph);
        AF_LT(3, n);
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < kHalves; ++hh)
#pragma unroll
          for (int kk = 0; kk < kLinChunk / 16; ++kk)
            mma_ss(tmem + kColH + hh * kLinVB,
                   make_sdesc(ka + hh * 2 * (kLinChunk * 128) + kk * 2048, kLinChunk * 128, 1024),
                   make_sdesc(aVw + kk * 2048, 16384, 1024), id_h, (n > 0 || kk > 0));
        mma_commit(h_full);
        mma_commit(&empty[st]);  // Q, K of this chunk: last read by the state update
        mbar_wait(p_ready, ph);
        mbar_wait(&vfull[sv], (n / kVSt) & 1);
        AF_LT(2, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kLinChunk / 16; ++kk)
          mma_ts(tmem + kColOI + ph * kLinVB, tmem + kColS + split_col_lin(kk),
                 make_sdesc(va + kk * 2048, 16384, 1024), id_oi, kk > 0);
        mma_commit(&oi_full[ph]);
        mma_commit(&vempty[sv]);  // V: last read by O I (the row warps' Vw copy came earlier)
      }
    }
  } else if (warp >= 8) {
    // ───────────── output warps: O = s_out (OI + cp QH) of chunk n, 64 columns per row ─────────
    const int wq = warp - 8;
    const int r = wq * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    for (int n = 0; n < nchunks; ++n) {
      const int c = kReverse ? nchunks - 1 - n : n;
      const int t = c * kLinChunk + r;
      const uint32_t ph = n & 1;
      const bool live = t < p.seq;
      LIN_IDLE_WAIT(&cp_ready[ph], (n >> 1) & 1);
      const float cp = sCp[ph * kLinChunk + r];
      const float rs = (p.o_rowscale.ptr != nullptr && live) ? p.o_rowscale.at(b, h, t) : 1.0f;
      LIN_IDLE_WAIT(&oi_full[ph], (n >> 1) & 1);
      if (warp == 8 && lane_id() == 0) AF_LT(9, n);
      tc_fence_after();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        const int col0 = vb * kLinVB + half * 32;
        __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o) + b * p.o_sb + h * p.o_sh +
                              static_cast<int64_t>(live ? t : 0) * p.o_ss + col0;
        uint32_t oi[32], qh[32];
        tmem_ld32(tmem + lane_base + kColOI + ph * kLinVB + half * 32, oi);
        tmem_ld32(tmem + lane_base + kColQH + ph * kLinVB + half * 32, qh);
        tmem_ld_wait();
        if (half == 1) {  // both halves read: release the OI / QH buffers and sCp[ph]
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&oi_empty[ph]);
        }
        float ov[32];
#pragma unroll
        for (int e = 0; e < 32; ++e)
          ov[e] = p.out_scale * fmaf(cp, __uint_as_float(qh[e]), __uint_as_float(oi[e]));
        if (live) {
          uint4* d4 = reinterpret_cast<uint4*>(orow);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            d4[v] = make_uint4(pack_bf16(rs * ov[v * 8 + 0], rs * ov[v * 8 + 1]),
                               pack_bf16(rs * ov[v * 8 + 2], rs * ov[v * 8 + 3]),
                               pack_bf16(rs * ov[v * 8 + 4], rs * ov[v * 8 + 5]),
                               pack_bf16(rs * ov[v * 8 + 6], rs * ov[v * 8 + 7]));
          if (p.dot_x != nullptr) {
            const uint4* x4 = reinterpret_cast<const uint4*>(
                reinterpret_cast<const __nv_bfloat16*>(p.dot_x) + b * p.x_sb + h * p.x_sh +
                static_cast<int64_t>(t) * p.x_ss + col0);
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
            const int64_t at =
                (vb * 2 + half) * rows + (static_cast<int64_t>(b) * p.heads + h) * p.seq + t;
            p.dot[at] = dotacc;
            if (p.dot2_x != nullptr) {
              const uint4* y4 = reinterpret_cast<const uint4*>(
                  reinterpret_cast<const __nv_bfloat16*>(p.dot2_x) + b * p.x_sb + h * p.x_sh +
                  static_cast<int64_t>(t) * p.x_ss + col0);
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
      if (warp == 8 && lane_id() == 0) AF_LT(10, n);
    }
  } else {
    // ───────────── chunk-row warps: two per TMEM lane quarter, column halves ─────────────
    const int wq = warp % 4;
    const int half = warp / 4;
    const int r = wq * 32 + static_cast<int>(lane_id());
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    for (int n = 0; n < nchunks; ++n) {
      const int c = kReverse ? nchunks - 1 - n : n;
      const int t = c * kLinChunk + r;
      const uint32_t ph = n & 1;
      const bool live = t < p.seq;
      (void)live;
      // (a) the producer warp's scan of this chunk (shared [n % 2] arrays)
      const float* sL = sLb + ph * kLinChunk;
      const float* sU = sUb + ph * kLinChunk;
      const float* sEc = sEcb + ph * kLinChunk;
      LIN_IDLE_WAIT(&scan_ready[ph], (n >> 1) & 1);
      if (threadIdx.x == 0) AF_LT(14, n);
      if (threadIdx.x == 0) AF_LT(18, n);
      const float l_r = sL[r];
      const float l_last = sL[kLinChunk - 1];
      const float g = exp2f(l_last);
      const float cp = kReverse ? exp2f(l_last - l_r) : exp2f(l_r);
      const float wgt = sU[r] * (kReverse ? exp2f(l_r) : exp2f(l_last - l_r));
      if (threadIdx.x == 0) AF_LT(19, n);
      if (half == 0) {  // hand cp to the output warps (sCp[ph] is free once chunk n-2 is out)
        if (n >= 2) mbar_wait(&oi_empty[ph], ((n >> 1) - 1) & 1);
        sCp[ph * kLinChunk + r] = cp;
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&cp_ready[ph]);
      }
      if (threadIdx.x == 0) AF_LT(4, n);
      // (b) Vw = diag(w * u_scale) V (this half's 4 granules; the previous state update is done)
      const int sv = n % kVSt;
      mbar_wait(&vfull[sv], (n / kVSt) & 1);
      if (threadIdx.x == 0) AF_LT(13, n);
#pragma unroll
      for (int gq = 0; gq < 4; ++gq) {
        const int gidx = half * 4 + gq;
        uint4 vv = *swz_row(sV + sv * L::kVBytes, r, gidx);
        uint32_t* e = reinterpret_cast<uint32_t*>(&vv);
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2)
          e[q2] = pack_bf16(bf16_lo_(e[q2]) * wgt, bf16_hi_(e[q2]) * wgt);
        *swz_row(sVw, r, gidx) = vv;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(vw_ready);
      if (threadIdx.x == 0) AF_LT(5, n);
      // (d) H <- g H for this half's 32 of every 64 state columns (chunk 0: the update MMA
      //     overwrites instead of accumulating)
      if (n > 0) {
#pragma unroll
        for (int hh = 0; hh < kHalves; ++hh) {
          uint32_t hr[32];
          const uint32_t col = tmem + lane_base + kColH + hh * kLinVB + half * 32;
          tmem_ld32(col, hr);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) hr[e] = __float_as_uint(__uint_as_float(hr[e]) * g);
          tmem_st32(col, hr);
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(h_scaled);
      if (threadIdx.x == 0) AF_LT(6, n);
      // (c) P = S o D o u_scale over this half's 64 key columns
      mbar_wait(s_full, ph);
      if (threadIdx.x == 0) AF_LT(7, n);
      tc_fence_after();
      {
        uint32_t pk[32];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          // warp-uniform 32x32 sub-block class: rows [wq*32, +32) x key columns [u0, u0+32)
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
          if (sFac[ph * 4 + (u0 >> 5)] != 0) {
            const float er = exp2f(kReverse ? sL[u0 + 31] - l_r : l_r - sL[u0]);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              const int u = u0 + e;
              const float4 c4 = *reinterpret_cast<const float4*>(sEc + u);
              const float cu[4] = {c4.x, c4.y, c4.z, c4.w};
              float pv[4];
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                const bool keep = all || (kReverse ? (u + x >= r) : (u + x <= r));
                pv[x] = keep ? __uint_as_float(sr[e + x]) * (er * cu[x]) : 0.0f;
              }
              pk[cc * 16 + e / 2] = pack_bf16(pv[0], pv[1]);
              pk[cc * 16 + e / 2 + 1] = pack_bf16(pv[2], pv[3]);
            }
            continue;
          }
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const int u = u0 + e;
            const float4 l4 = *reinterpret_cast<const float4*>(sL + u);
            const float4 u4 = *reinterpret_cast<const float4*>(sU + u);
            const float lu[4] = {l4.x, l4.y, l4.z, l4.w};
            const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
            float pv[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const bool keep = all || (kReverse ? (u + x >= r) : (u + x <= r));
              const float d = ex2(kReverse ? lu[x] - l_r : l_r - lu[x]) * uu[x];
              pv[x] = keep ? __uint_as_float(sr[e + x]) * d : 0.0f;
            }
            pk[cc * 16 + e / 2] = pack_bf16(pv[0], pv[1]);
            pk[cc * 16 + e / 2 + 1] = pack_bf16(pv[2], pv[3]);
          }
        }
        tmem_st32(tmem + lane_base + kColS + half * 64, pk);  // packed: see split_col_lin
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) {
        mbar_arrive(p_ready);
        mbar_arrive(&scan_free[ph]);  // this chunk's scan arrays read (last use: P)
      }
      if (threadIdx.x == 0) AF_LT(8, n);
      // (f) bf16 copy of the updated state (this half's columns) for the next chunk's Q H —
      //     after Q H of this chunk has read the previous copy
      mbar_wait(h_full, ph);
      mbar_wait(qh_full, ph);
      if (threadIdx.x == 0) AF_LT(11, n);
      tc_fence_after();
#pragma unroll
      for (int hh = 0; hh < kHalves; ++hh) {
        const int dk = hh * 128 + r;
        uint32_t hr[32];
        tmem_ld32(tmem + lane_base + kColH + hh * kLinVB + half * 32, hr);
        tmem_ld_wait();
#pragma unroll
        for (int gq = 0; gq < 4; ++gq)
          *swz_row(sHb, dk, half * 4 + gq) = make_uint4(
              pack_bf16(__uint_as_float(hr[gq * 8 + 0]), __uint_as_float(hr[gq * 8 + 1])),
              pack_bf16(__uint_as_float(hr[gq * 8 + 2]), __uint_as_float(hr[gq * 8 + 3])),
              pack_bf16(__uint_as_float(hr[gq * 8 + 4]), __uint_as_float(hr[gq * 8 + 5])),
              pack_bf16(__uint_as_float(hr[gq * 8 + 6]), __uint_as_float(hr[gq * 8 + 7])));
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(hb_ready);
      if (threadIdx.x == 0) AF_LT(12, n);
      if (!kReverse && p.final_state != nullptr && n == nchunks - 1) {
        // the state after the last chunk (run_step_recurrent's h_S): fp32 [dk][dv] rows, this
        // half's 32 columns of the CTA's 64-column value block
#pragma unroll
        for (int hh = 0; hh < kHalves; ++hh) {
          const int dk = hh * 128 + r;
          uint32_t hr[32];
          tmem_ld32(tmem + lane_base + kColH + hh * kLinVB + half * 32, hr);
          tmem_ld_wait();
          float4* dst = reinterpret_cast<float4*>(
              p.final_state + ((static_cast<int64_t>(b) * p.heads + h) * p.dqk + dk) * p.dv +
              vb * kLinVB + half * 32);
#pragma unroll
          for (int v4 = 0; v4 < 8; ++v4)
            dst[v4] = make_float4(__uint_as_float(hr[v4 * 4]), __uint_as_float(hr[v4 * 4 + 1]),
                                  __uint_as_float(hr[v4 * 4 + 2]), __uint_as_float(hr[v4 * 4 + 3]));
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Per-step gradients (SURVEY A.4 restated):  d log a_t = sum_{s>=t} (dq_dot_s - dk_dot_s)
// where dq_dot = Qm . dQm, dk_dot = Km . dKm over the same bf16 gated keys the passes used (the
// two sums nearly cancel; a dot over u k instead of bf16(u k) measured 5 % off the oracle), and
// kdot_raw = k . dKm over the raw keys (when the key gate is not also a decay factor).  One block
// per (b, h) sequence writes d log a_t and the gate's dot (both [B, H, S] fp32);
// step_grad_reduce_multi_kernel then forms d fac_f = d log a / fac_f and d gate = kdot_raw (k_mod =
// k * gate: dL/dgate = k . dKm, no division — finite at gate = 0; else dk_dot / gate) and sums
// broadcast axes in a fixed order — no atomics, bitwise deterministic.  A decay factor of exactly
// 0 gives a non-finite d fac at that step (d log a / 0; the unrolled reference differentiates
// the product itself).
// One block per (b, h) sequence: each thread sums a contiguous run of steps, a block-wide
// exclusive suffix scan of the run totals (warp shuffles + one smem pass) hands every run its
// carry, then the run is re-walked writing d log a_t and the gate's dot (a one-warp-per-32-steps
// form with 256 threads took 0.13 ms at cfg5b: the serial runs were 32 steps of 8 strided loads).
constexpr int kStepGradThreads = 1024;
__global__ void __launch_bounds__(kStepGradThreads)
    linear_step_grads_kernel(const float* __restrict__ dq_dot, const float* __restrict__ dk_dot,
                             const float* __restrict__ kdot_raw, int slots, LinearParams p,
                             float* __restrict__ dloga_out, float* __restrict__ dkdot_out) {
  __shared__ float part[kStepGradThreads / 32];
  const int bh = blockIdx.x;
  const int64_t base = static_cast<int64_t>(bh) * p.seq;
  const int seq = p.seq;
  const int64_t rows = static_cast<int64_t>(p.batch) * p.heads * p.seq;
  auto dot = [&](const float* x, int t) {  // per-slot partials, summed in a fixed slot order
    float a = 0.0f;
    for (int sl = 0; sl < slots; ++sl) a += x[sl * rows + base + t];
    return a;
  };
  auto val = [&](int t) { return dot(dq_dot, t) - dot(dk_dot, t); };
  const int per = (seq + blockDim.x - 1) / blockDim.x;
  const int t0 = threadIdx.x * per;
  const int t1 = min(seq, t0 + per);
  float s = 0.0f;
  for (int t = t1 - 1; t >= t0; --t) s += val(t);
  // exclusive suffix sum of the run totals over the block (later threads = later steps)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = static_cast<int>(blockDim.x >> 5);
  float x = s;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float y = __shfl_down_sync(0xffffffffu, x, off);
    if (lane + off < 32) x += y;
  }
  if (lane == 0) part[w] = x;  // warp total
  __syncthreads();
  if (w == 0) {  // inclusive suffix scan of the warp totals
    float v = lane < nw ? part[lane] : 0.0f;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float y = __shfl_down_sync(0xffffffffu, v, off);
      if (lane + off < 32) v += y;
    }
    if (lane < nw) part[lane] = v;
  }
  __syncthreads();
  float acc = (x - s) + (w + 1 < nw ? part[w + 1] : 0.0f);  // every step after this run
  for (int t = t1 - 1; t >= t0; --t) {
    acc += val(t);
    dloga_out[base + t] = acc;
    if (dkdot_out != nullptr) dkdot_out[base + t] = dot(kdot_raw != nullptr ? kdot_raw : dk_dot, t);
  }
}

// out[b', h', t] += sum over the broadcast axes of out (stride 0) of val[b, h, t] / div(b, h, t)
// (div.ptr null: val itself),
// in ascending (b, h) order.  val is [B, H, S] fp32; one thread per output element.
// The per-step reductions (out[b, h, t] += sum over broadcast axes of val / div, fixed order) — up
// to three in one launch (decay factors and the gate of one call; a
// gate that is also a decay factor writes the same tensor twice — in the same thread, in job
// order).  Every job's output must share one broadcast pattern (else separate launches).
struct StepReduceJob {
  const float* val;
  StepTensor div, out;
};
struct StepReduceJobs {
  StepReduceJob job[3];
  int n;
};
__global__ void step_grad_reduce_multi_kernel(StepReduceJobs jobs, int batch, int heads, int seq) {
  const StepTensor& o0 = jobs.job[0].out;
  const int nb = o0.sb == 0 ? 1 : batch, nh = o0.sh == 0 ? 1 : heads;
  const int64_t total = static_cast<int64_t>(nb) * nh * seq;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= total) return;
  const int t = static_cast<int>(gid % seq);
  const int hh = static_cast<int>((gid / seq) % nh);
  const int bb = static_cast<int>(gid / (static_cast<int64_t>(seq) * nh));
  for (int j = 0; j < jobs.n; ++j) {
    const StepReduceJob& jb = jobs.job[j];
    float acc = 0.0f;
    for (int b = (o0.sb == 0 ? 0 : bb); b < (o0.sb == 0 ? batch : bb + 1); ++b)
      for (int h = (o0.sh == 0 ? 0 : hh); h < (o0.sh == 0 ? heads : hh + 1); ++h)
        acc += jb.div.ptr != nullptr
                   ? jb.val[(static_cast<int64_t>(b) * heads + h) * seq + t] / jb.div.at(b, h, t)
                   : jb.val[(static_cast<int64_t>(b) * heads + h) * seq + t];
    float* dst = const_cast<float*>(jb.out.ptr) + bb * jb.out.sb + hh * jb.out.sh + t * jb.out.ss;
    *dst += acc;
  }
}

// Km = bf16(k * gate): the backward uses one rounded copy of the gated keys in every pass so the
// two dot terms of d log a cancel consistently (folding the gate into P / Vw instead rounds the
// passes differently and loses ~2 digits in the cancellation).
// Each thread scales kGkVec 16-byte chunks of one key row (independent loads in flight: one chunk
// per thread ran at 4.4 TB/s on cfg5b's 268 MB of keys).
constexpr int kGkVec = 4;
__global__ void gate_keys_kernel(const __nv_bfloat16* __restrict__ k, int64_t sb, int64_t sh,
                                 int64_t ss, StepTensor gate, int heads, int seq, int dk,
                                 __nv_bfloat16* __restrict__ out, int64_t total_rows) {
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int per_row = dk >= 8 * kGkVec ? dk / (8 * kGkVec) : 1;  // threads per row
  const int64_t row = gid / per_row;
  if (row >= total_rows) return;
  const int c0 = static_cast<int>(gid % per_row) * 8;  // chunk j at c0 + 8 * per_row * j
  const int t = static_cast<int>(row % seq);
  const int64_t bh = row / seq;
  const int b = static_cast<int>(bh / heads), h = static_cast<int>(bh % heads);
  const float g = gate.at(b, h, t);
  const __nv_bfloat16* src = k + b * sb + h * sh + t * ss;
  uint4 x[kGkVec];
#pragma unroll
  for (int j = 0; j < kGkVec; ++j)
    x[j] = c0 + 8 * per_row * j < dk ? *reinterpret_cast<const uint4*>(src + c0 + 8 * per_row * j)
                                     : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
  for (int j = 0; j < kGkVec; ++j) {
    const uint32_t* e = reinterpret_cast<const uint32_t*>(&x[j]);
    uint4 y;
    uint32_t* o = reinterpret_cast<uint32_t*>(&y);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = pack_bf16(bf16_lo_(e[i]) * g, bf16_hi_(e[i]) * g);
    if (c0 + 8 * per_row * j < dk)
      *reinterpret_cast<uint4*>(out + row * dk + c0 + 8 * per_row * j) = y;
  }
}

}  // namespace af
