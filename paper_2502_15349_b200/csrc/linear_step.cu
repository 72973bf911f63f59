// K4s — single-token step of the linear (recurrent) template for generation: the body of
// attnforge `engine.run_step_recurrent` (engine.py:539-547) for one new token t, on a carried fp32
// state (e.g. the final_state of af_linear_fwd over the prompt):
//   h <- a_t h + (k_t * gate_t)^T v_t ,   o_t = q_scale * q_t h
// HBM-bound (the state is read and written once per step); one CTA per (b, h), one thread per
// value column, the state rows streamed with coalesced fp32 loads / stores.
#include <cuda_bf16.h>

#include <algorithm>

#include "host_common.h"
#include "sm100.cuh"

namespace af {
namespace {

// per-step fp32 tensor with element strides [b, h, s] (0 = broadcast axis)
struct StepTensor {
  const float* ptr;
  int64_t sb, sh, ss;
  AF_DEVICE float at(int b, int h, int t) const { return ptr[b * sb + h * sh + t * ss]; }
};

struct StepParams {
  int heads, dk, dv;
  float q_scale, log_const;
  int nfac;
  StepTensor fac[2];
  StepTensor gate;
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  int64_t q_sb, q_sh, k_sb, k_sh, v_sb, v_sh, o_sb, o_sh;
  __nv_bfloat16* o;
  float* state;  // [B, H, dk, dv] fp32, updated in place
};

__global__ void linear_step_kernel(const StepParams p) {
  extern __shared__ float sh[];  // q [dk] | k*gate [dk]
  const int bh = blockIdx.x;
  const int b = bh / p.heads, h = bh % p.heads;
  float a = __expf(p.log_const);
  for (int f = 0; f < p.nfac; ++f) a *= p.fac[f].at(b, h, 0);
  const float u = (p.gate.ptr != nullptr) ? p.gate.at(b, h, 0) : 1.0f;
  for (int i = threadIdx.x; i < p.dk; i += blockDim.x) {
    sh[i] = __bfloat162float(p.q[b * p.q_sb + h * p.q_sh + i]);
    sh[p.dk + i] = __bfloat162float(p.k[b * p.k_sb + h * p.k_sh + i]) * u;
  }
  __syncthreads();
  float* st = p.state + static_cast<int64_t>(bh) * p.dk * p.dv;
  for (int j = threadIdx.x; j < p.dv; j += blockDim.x) {
    const float vj = __bfloat162float(p.v[b * p.v_sb + h * p.v_sh + j]);
    float acc = 0.0f;
#pragma unroll 4
    for (int i = 0; i < p.dk; ++i) {
      const float s = fmaf(a, st[static_cast<int64_t>(i) * p.dv + j], sh[p.dk + i] * vj);
      st[static_cast<int64_t>(i) * p.dv + j] = s;
      acc = fmaf(sh[i], s, acc);
    }
    p.o[b * p.o_sb + h * p.o_sh + j] = __float2bfloat16_rn(p.q_scale * acc);
  }
}

StepTensor step_of(const float* ptr, const int64_t* st) {
  StepTensor t{};
  t.ptr = ptr;
  if (ptr != nullptr) {
    t.sb = st[0];
    t.sh = st[1];
    t.ss = st[2];
  }
  return t;
}

}  // namespace
}  // namespace af

extern "C" int af_linear_step(const af_linear_desc* d, const void* q, const void* k,
                              const void* v, float* state, void* o, void* stream) {
  using namespace af;
  AF_REQUIRE(d != nullptr && state != nullptr, AF_ERR_INPUT, "null descriptor / state");
  AF_REQUIRE(d->seq == 1, AF_ERR_SHAPE, "af_linear_step takes one token (seq = %d)", d->seq);
  AF_REQUIRE(d->batch >= 1 && d->heads >= 1 && d->d_k >= 1 && d->d_v >= 1 && d->d_k <= 4096,
             AF_ERR_INPUT, "bad dims");
  AF_REQUIRE(d->n_decay_factors >= 0 && d->n_decay_factors <= 2, AF_ERR_UNSUPPORTED,
             "at most two per-step decay factors");
  StepParams p{};
  p.heads = d->heads;
  p.dk = d->d_k;
  p.dv = d->d_v;
  p.q_scale = d->q_scale;
  p.log_const = d->log_decay_const;
  p.nfac = d->n_decay_factors;
  for (int f = 0; f < p.nfac; ++f) p.fac[f] = step_of(d->decay_factor[f], d->decay_factor_stride[f]);
  p.gate = step_of(d->key_gate, d->key_gate_stride);
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.k = static_cast<const __nv_bfloat16*>(k);
  p.v = static_cast<const __nv_bfloat16*>(v);
  p.q_sb = d->q_stride[0]; p.q_sh = d->q_stride[1];
  p.k_sb = d->k_stride[0]; p.k_sh = d->k_stride[1];
  p.v_sb = d->v_stride[0]; p.v_sh = d->v_stride[1];
  p.o_sb = d->o_stride[0]; p.o_sh = d->o_stride[1];
  p.o = static_cast<__nv_bfloat16*>(o);
  p.state = state;
  const int threads = std::min(1024, ((d->d_v + 31) / 32) * 32);
  ::af::note_launch();
  linear_step_kernel<<<d->batch * d->heads, threads, 2 * d->d_k * sizeof(float),
                       reinterpret_cast<cudaStream_t>(stream)>>>(p);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}
