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

constexpr int kRows = 128;  // query rows per CTA (one per thread)
constexpr int kKeys = 32;   // keys staged per block

__device__ __forceinline__ bool kept32(const MaskParams& m, int i, int j, int seq_k) {
  bool k = j < seq_k;
  if (m.causal) k = k && (j <= i + m.diag_offset);
  if (m.window > 0) k = k && (i + m.diag_offset - j < m.window);
  return k;
}

template <int D, int DV>
__global__ void __launch_bounds__(kRows) parallel_fwd_f32_kernel(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    af_parallel_desc d, float* __restrict__ o, float* __restrict__ lse) {
  __shared__ float sk[kKeys][D];
  __shared__ float sv[kKeys][DV];
  const int bh = blockIdx.y;
  const int b = bh / d.heads_q, h = bh % d.heads_q;
  const int hk = h / (d.heads_q / d.heads_kv);
  const int i = blockIdx.x * kRows + threadIdx.x;
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

  for (int j0 = lo; j0 < hi; j0 += kKeys) {
    __syncthreads();
    for (int e = threadIdx.x; e < kKeys * D; e += kRows) {
      const int r = e / D, c = e % D, j = j0 + r;
      sk[r][c] = (j < d.seq_k) ? k[b * d.k_stride[0] + hk * d.k_stride[1] + static_cast<int64_t>(j) * d.k_stride[2] + c] : 0.f;
    }
    for (int e = threadIdx.x; e < kKeys * DV; e += kRows) {
      const int r = e / DV, c = e % DV, j = j0 + r;
      sv[r][c] = (j < d.seq_k) ? v[b * d.v_stride[0] + hk * d.v_stride[1] + static_cast<int64_t>(j) * d.v_stride[2] + c] : 0.f;
    }
    __syncthreads();
    float s[kKeys];
#pragma unroll 4
    for (int r = 0; r < kKeys; ++r) {
      float dot = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) dot = fmaf(qr[c], sk[r][c], dot);
      s[r] = dot;
    }
    if (d.family == AF_FAMILY_SOFTMAX) {
      float bmax = -INFINITY;
      for (int r = 0; r < kKeys; ++r) {
        if (d.cap_b != 0.f) s[r] = d.cap_a * tanhf(d.cap_b * s[r]);  // soft-cap (scaled logits)
        if (!kept32(m, i, j0 + r, d.seq_k)) s[r] = -INFINITY;
        bmax = fmaxf(bmax, s[r]);
      }
      const float m_new = fmaxf(m_run, bmax);
      const float rsc = (m_new == -INFINITY) ? 1.f : expf(m_run - m_new);
      float lsum = 0.f;
      for (int r = 0; r < kKeys; ++r) {
        s[r] = (m_new == -INFINITY) ? 0.f : expf(s[r] - m_new);
        lsum += s[r];
      }
      l_run = rsc * l_run + lsum;
      m_run = m_new;
#pragma unroll
      for (int c = 0; c < DV; ++c) acc[c] *= rsc;
    } else if (d.family == AF_FAMILY_ABSSUM) {
      // retention-parallel: s * gamma^(i-j) on the band, row abs-sum in l_run (slope = log2 g)
      for (int r = 0; r < kKeys; ++r) {
        const int j = j0 + r;
        const float z = kept32(m, i, j, d.seq_k) ? s[r] * exp2f(static_cast<float>(i - j) * slope)
                                                 : 0.f;
        l_run += fabsf(z);
        s[r] = z;
      }
    } else {
      for (int r = 0; r < kKeys; ++r) {
        const int j = j0 + r;
        float z = s[r] - slope * static_cast<float>(i - j) + d.bias;
        if (d.act == AF_ACT_SIGMOID) z = 1.f / (1.f + expf(-z));
        else if (d.act == AF_ACT_RELU) z = fmaxf(z, 0.f);
        else if (d.act == AF_ACT_RELU2) z = fmaxf(z, 0.f) * fmaxf(z, 0.f);
        s[r] = kept32(m, i, j, d.seq_k) ? z : 0.f;
      }
    }
#pragma unroll 4
    for (int r = 0; r < kKeys; ++r) {
#pragma unroll
      for (int c = 0; c < DV; ++c) acc[c] = fmaf(s[r], sv[r][c], acc[c]);
    }
  }
  if (!live) return;
  float* op = o + b * d.o_stride[0] + h * d.o_stride[1] + static_cast<int64_t>(i) * d.o_stride[2];
  if (d.family == AF_FAMILY_SOFTMAX) {
#pragma unroll
    for (int c = 0; c < DV; ++c) op[c] = (l_run == 0.f) ? 0.f : acc[c] / l_run;
    if (lse != nullptr)
      lse[(static_cast<int64_t>(b) * d.heads_q + h) * d.seq_q + i] =
          (l_run == 0.f) ? -INFINITY : m_run + logf(l_run);
  } else if (d.family == AF_FAMILY_ABSSUM) {
    const float inv = (d.cap_a != 0.f) ? 1.f / fmaxf(l_run, 1.f) : 1.f;
#pragma unroll
    for (int c = 0; c < DV; ++c) op[c] = acc[c] * inv;
    if (lse != nullptr) lse[(static_cast<int64_t>(b) * d.heads_q + h) * d.seq_q + i] = l_run;
  } else {
#pragma unroll
    for (int c = 0; c < DV; ++c) op[c] = acc[c];
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
    kern<<<grid, kRows, 0, s>>>(static_cast<const float*>(q), static_cast<const float*>(k),
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
