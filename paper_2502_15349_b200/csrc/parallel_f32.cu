// fp32 parallel-template forward (cfg1 parity case: fp32 in/out, 1e-5 vs the f64 oracle).
//
// tcgen05 has no fp32-input MMA (kind::tf32 truncates to 10 mantissa bits), so the fp32 path runs
// exact FFMA: one thread owns one query row (q and the output accumulator live in registers),
// key/value blocks of 32 rows are staged in shared memory and the online protocol of
// engine.run_tiled_parallel (engine.py:465-500) runs per block with IEEE expf / division.
#include "host_common.h"
#include "params.h"

namespace af {
namespace {

// Each query row is shared by the kSplit lanes of a warp, which take interleaved keys of every
// staged block and merge their (max, sum, accumulator) states at the end: a row-per-thread form
// ran 16 CTAs of 128 threads at cfg1 (B1 H4 S512) — 0.41 ms of serial per-thread chains on 16 of
// 148 SMs; 8 lanes per row 0.078 ms; a warp per row (512 CTAs) see DESIGN §3.
constexpr int kSplit = 32;                 // threads per query row (a warp)
constexpr int kThreads = 128;
constexpr int kRows = kThreads / kSplit;   // query rows per CTA
// keys staged per block: 64 (half the block iterations, each paying a global-load latency) while
// the padded K and V blocks fit the 48 KB static shared memory, else 32
template <int D, int DV>
constexpr int keys_per_block() { return (D + 1 + DV + 1) * 64 * 4 <= 48 * 1024 ? 64 : 32; }

__device__ __forceinline__ bool kept32(const MaskParams& m, int i, int j, int seq_k) {
  bool k = j < seq_k;
  if (m.causal) k = k && (j <= i + m.diag_offset);
  if (m.window > 0) k = k && (i + m.diag_offset - j < m.window);
  return k;
}

template <int D, int DV>
__global__ void __launch_bounds__(kThreads) parallel_fwd_f32_kernel(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    af_parallel_desc d, float* __restrict__ o, float* __restrict__ lse) {
  // rows padded by one word: the lanes of a row read 32 different key rows at the same column
  // (unpadded, a power-of-two row stride put them all in one bank)
  constexpr int kKeys = keys_per_block<D, DV>();
  __shared__ float sk[kKeys][D + 1];
  __shared__ float sv[kKeys][DV + 1];
  const int bh = blockIdx.y;
  const int b = bh / d.heads_q, h = bh % d.heads_q;
  const int hk = h / (d.heads_q / d.heads_kv);
  const int sp = static_cast<int>(threadIdx.x) % kSplit;  // this thread's key phase
  const int i = blockIdx.x * kRows + static_cast<int>(threadIdx.x) / kSplit;
  const bool live = i < d.seq_q;
  const MaskParams m{d.causal, d.diag_offset, d.window};

  float qr[D];
  const float* qp = q + b * d.q_stride[0] + h * d.q_stride[1] + static_cast<int64_t>(live ? i : 0) * d.q_stride[2];
#pragma unroll
  for (int c = 0; c < D; ++c) qr[c] = qp[c] * d.scale;  // q_mod folded (q / sqrt(dimqk))
  float acc[DV];
#pragma unroll
  for (int c = 0; c < DV; ++c) acc[c] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  const float slope = (d.slope != nullptr) ? d.slope[h] : 0.f;

  // Key range any row of the CTA can see.
  const int r0 = blockIdx.x * kRows, r1 = min(d.seq_q, r0 + kRows);
  int hi = d.seq_k, lo = 0;
  if (d.causal) hi = min(hi, r1 - 1 + d.diag_offset + 1);
  if (d.window > 0) lo = max(0, r0 + d.diag_offset - d.window + 1);
  lo = (lo / kKeys) * kKeys;

  constexpr int kPer = kKeys / kSplit;  // keys of a block per thread: r = sp + kSplit * t
  const bool vec = ((d.k_stride[0] | d.k_stride[1] | d.k_stride[2] | d.v_stride[0] |
                     d.v_stride[1] | d.v_stride[2]) % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) % 16 == 0);
  for (int j0 = lo; j0 < hi; j0 += kKeys) {
    __syncthreads();
    if (D % 4 == 0 && DV % 4 == 0 && vec) {  // 16-byte loads
      for (int e = threadIdx.x; e < kKeys * D / 4; e += kThreads) {
        const int r = e / (D / 4), c = (e % (D / 4)) * 4, j = j0 + r;
        const float4 x = (j < d.seq_k) ? *reinterpret_cast<const float4*>(
                                             k + b * d.k_stride[0] + hk * d.k_stride[1] +
                                             static_cast<int64_t>(j) * d.k_stride[2] + c)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        sk[r][c] = x.x;
        sk[r][c + 1] = x.y;
        sk[r][c + 2] = x.z;
        sk[r][c + 3] = x.w;
      }
      for (int e = threadIdx.x; e < kKeys * DV / 4; e += kThreads) {
        const int r = e / (DV / 4), c = (e % (DV / 4)) * 4, j = j0 + r;
        const float4 x = (j < d.seq_k) ? *reinterpret_cast<const float4*>(
                                             v + b * d.v_stride[0] + hk * d.v_stride[1] +
                                             static_cast<int64_t>(j) * d.v_stride[2] + c)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        sv[r][c] = x.x;
        sv[r][c + 1] = x.y;
        sv[r][c + 2] = x.z;
        sv[r][c + 3] = x.w;
      }
    } else {
      for (int e = threadIdx.x; e < kKeys * D; e += kThreads) {
        const int r = e / D, c = e % D, j = j0 + r;
        sk[r][c] = (j < d.seq_k) ? k[b * d.k_stride[0] + hk * d.k_stride[1] + static_cast<int64_t>(j) * d.k_stride[2] + c] : 0.f;
      }
      for (int e = threadIdx.x; e < kKeys * DV; e += kThreads) {
        const int r = e / DV, c = e % DV, j = j0 + r;
        sv[r][c] = (j < d.seq_k) ? v[b * d.v_stride[0] + hk * d.v_stride[1] + static_cast<int64_t>(j) * d.v_stride[2] + c] : 0.f;
      }
    }
    __syncthreads();
    float s[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int r = sp + kSplit * t;
      float dot = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) dot = fmaf(qr[c], sk[r][c], dot);
      s[t] = dot;
    }
    if (d.family == AF_FAMILY_SOFTMAX) {
      float bmax = -INFINITY;
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        if (d.cap_b != 0.f) s[t] = d.cap_a * tanhf(d.cap_b * s[t]);  // soft-cap (scaled logits)
        if (!kept32(m, i, j0 + sp + kSplit * t, d.seq_k)) s[t] = -INFINITY;
        bmax = fmaxf(bmax, s[t]);
      }
      const float m_new = fmaxf(m_run, bmax);
      const float rsc = (m_new == -INFINITY) ? 1.f : expf(m_run - m_new);
      float lsum = 0.f;
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        s[t] = (m_new == -INFINITY) ? 0.f : expf(s[t] - m_new);
        lsum += s[t];
      }
      l_run = rsc * l_run + lsum;
      m_run = m_new;
#pragma unroll
      for (int c = 0; c < DV; ++c) acc[c] *= rsc;
    } else if (d.family == AF_FAMILY_ABSSUM) {
      // retention-parallel: s * gamma^(i-j) on the band, row abs-sum in l_run (slope = log2 g)
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const int j = j0 + sp + kSplit * t;
        const float z = kept32(m, i, j, d.seq_k) ? s[t] * exp2f(static_cast<float>(i - j) * slope)
                                                 : 0.f;
        l_run += fabsf(z);
        s[t] = z;
      }
    } else {
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const int j = j0 + sp + kSplit * t;
        float z = s[t] - slope * static_cast<float>(i - j) + d.bias;
        if (d.act == AF_ACT_SIGMOID) z = 1.f / (1.f + expf(-z));
        else if (d.act == AF_ACT_RELU) z = fmaxf(z, 0.f);
        else if (d.act == AF_ACT_RELU2) z = fmaxf(z, 0.f) * fmaxf(z, 0.f);
        s[t] = kept32(m, i, j, d.seq_k) ? z : 0.f;
      }
    }
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int r = sp + kSplit * t;
#pragma unroll
      for (int c = 0; c < DV; ++c) acc[c] = fmaf(s[t], sv[r][c], acc[c]);
    }
  }
  // merge the kSplit partial states of the row (butterfly over the row's consecutive lanes:
  // every lane ends with the row's totals)
  if (d.family == AF_FAMILY_SOFTMAX) {
    float m_row = m_run;
#pragma unroll
    for (int off = 1; off < kSplit; off <<= 1)
      m_row = fmaxf(m_row, __shfl_xor_sync(0xffffffffu, m_row, off));
    const float f = (m_run == -INFINITY) ? 0.f : expf(m_run - m_row);
    l_run *= f;
#pragma unroll
    for (int c = 0; c < DV; ++c) acc[c] *= f;
    m_run = m_row;
  }
#pragma unroll
  for (int off = 1; off < kSplit; off <<= 1) {
    l_run += __shfl_xor_sync(0xffffffffu, l_run, off);
#pragma unroll
    for (int c = 0; c < DV; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], off);
  }
  if (!live) return;
  // each of the row's threads writes DV / kSplit of its columns (DV >= kSplit, else thread 0)
  constexpr int kCols = DV >= kSplit ? DV / kSplit : DV;
  const int c0 = DV >= kSplit ? sp * kCols : 0;
  if (DV < kSplit && sp != 0) return;
  float* op = o + b * d.o_stride[0] + h * d.o_stride[1] + static_cast<int64_t>(i) * d.o_stride[2];
  float scale = 1.f;
  if (d.family == AF_FAMILY_SOFTMAX) scale = (l_run == 0.f) ? 0.f : 1.f;
  else if (d.family == AF_FAMILY_ABSSUM) scale = (d.cap_a != 0.f) ? 1.f / fmaxf(l_run, 1.f) : 1.f;
#pragma unroll
  for (int c = 0; c < DV; ++c) {
    if (c < c0 || c >= c0 + kCols) continue;
    if (d.family == AF_FAMILY_SOFTMAX)
      op[c] = (l_run == 0.f) ? 0.f : acc[c] / l_run;
    else
      op[c] = acc[c] * scale;
  }
  if (sp == 0 && lse != nullptr) {
    if (d.family == AF_FAMILY_SOFTMAX)
      lse[(static_cast<int64_t>(b) * d.heads_q + h) * d.seq_q + i] =
          (l_run == 0.f) ? -INFINITY : m_run + logf(l_run);
    else if (d.family == AF_FAMILY_ABSSUM)
      lse[(static_cast<int64_t>(b) * d.heads_q + h) * d.seq_q + i] = l_run;
  }
}

}  // namespace
}  // namespace af

extern "C" int af_parallel_fwd_f32(const af_parallel_desc* d, const void* q, const void* k,
                                   const void* v, void* o, float* lse, void* stream) {
  using namespace af;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dim3 grid((d->seq_q + kRows - 1) / kRows, d->batch * d->heads_q);
  auto args = [&](auto kern) {
    ::af::note_launch();
    kern<<<grid, kThreads, 0, s>>>(static_cast<const float*>(q), static_cast<const float*>(k),
                                static_cast<const float*>(v), *d, static_cast<float*>(o), lse);
  };
  if (d->d_qk == 64 && d->d_v == 64) args(parallel_fwd_f32_kernel<64, 64>);
  else if (d->d_qk == 128 && d->d_v == 128) args(parallel_fwd_f32_kernel<128, 128>);
  else if (d->d_qk == 32 && d->d_v == 32) args(parallel_fwd_f32_kernel<32, 32>);
  else if (d->d_qk == 16 && d->d_v == 16) args(parallel_fwd_f32_kernel<16, 16>);
  else if (d->d_qk == 8 && d->d_v == 8) args(parallel_fwd_f32_kernel<8, 8>);
  else if (d->d_qk == 4 && d->d_v == 4) args(parallel_fwd_f32_kernel<4, 4>);
  else {
    set_error("fp32 parallel forward: head dims (%d, %d) not instantiated", d->d_qk, d->d_v);
    return AF_ERR_UNSUPPORTED;
  }
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}
