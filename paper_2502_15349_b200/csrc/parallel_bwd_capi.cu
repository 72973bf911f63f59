// C-ABI entry points of the parallel-template backward: workspace sizing, preprocess (row
// statistics), the K2 main kernel and the dQ fp32 -> bf16 conversion, all stream-ordered.
#include "host_common.h"
#include "parallel_bwd.cuh"

namespace af {
int validate_parallel(const af_parallel_desc* d);
namespace {

inline int64_t pad_q(int seq_q) { return ((seq_q + kBlockM - 1) / kBlockM) * kBlockM; }

template <int D, int DV, int kFamily, int kAct>
int launch_bwd(const af_parallel_desc* d, const CUtensorMap& tq, const CUtensorMap& tk,
               const CUtensorMap& tv, const CUtensorMap& tdo, const ParallelBwdParams& p,
               const float* lse2, const float* delta, int seq_q_pad, cudaStream_t stream) {
  using L = BwdSmem<D, DV>;
  auto kern = parallel_bwd_kernel<D, DV, kFamily, kAct>;
  static bool attr_done = false;
  if (!attr_done) {
    AF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal));
    attr_done = true;
  }
  dim3 grid((d->seq_k + kBlockN - 1) / kBlockN, d->batch * d->heads_kv);
  kern<<<grid, 512, L::kTotal, stream>>>(tq, tk, tv, tdo, p, lse2, delta, seq_q_pad);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

template <int D, int DV>
int dispatch_bwd(const af_parallel_desc* d, const CUtensorMap& tq, const CUtensorMap& tk,
                 const CUtensorMap& tv, const CUtensorMap& tdo, const ParallelBwdParams& p,
                 const float* lse2, const float* delta, int pad, cudaStream_t s) {
  if (d->family == AF_FAMILY_SOFTMAX)
    return launch_bwd<D, DV, kFamilySoftmax, kActIdentity>(d, tq, tk, tv, tdo, p, lse2, delta, pad, s);
  switch (d->act) {
    case AF_ACT_SIGMOID: return launch_bwd<D, DV, kFamilyElementwise, kActSigmoid>(d, tq, tk, tv, tdo, p, lse2, delta, pad, s);
    case AF_ACT_RELU: return launch_bwd<D, DV, kFamilyElementwise, kActRelu>(d, tq, tk, tv, tdo, p, lse2, delta, pad, s);
    case AF_ACT_IDENTITY: return launch_bwd<D, DV, kFamilyElementwise, kActIdentity>(d, tq, tk, tv, tdo, p, lse2, delta, pad, s);
    default: break;
  }
  set_error("unknown activation %d", d->act);
  return AF_ERR_INPUT;
}

}  // namespace
}  // namespace af

extern "C" size_t af_parallel_bwd_workspace(const af_parallel_desc* d) {
  if (d == nullptr) return 0;
  const int64_t rows = static_cast<int64_t>(d->batch) * d->heads_q * af::pad_q(d->seq_q);
  return static_cast<size_t>(rows) * (static_cast<size_t>(d->d_qk) + 2) * sizeof(float);
}

extern "C" int af_parallel_bwd(const af_parallel_desc* d, const void* q, const void* k,
                               const void* v, const void* o, const float* lse, const void* dout,
                               void* dq, void* dk, void* dv, void* workspace,
                               size_t workspace_bytes, void* stream) {
  using namespace af;
  int st = validate_parallel(d);
  if (st != AF_OK) return st;
  AF_REQUIRE(d->dtype == AF_DTYPE_BF16, AF_ERR_UNSUPPORTED, "backward runs on bf16 inputs only");
  AF_REQUIRE(workspace_bytes >= af_parallel_bwd_workspace(d), AF_ERR_INPUT,
             "workspace too small (%zu < %zu)", workspace_bytes, af_parallel_bwd_workspace(d));
  AF_REQUIRE(d->family != AF_FAMILY_SOFTMAX || lse != nullptr, AF_ERR_INPUT,
             "softmax backward needs the forward LSE");
  const int pad = static_cast<int>(pad_q(d->seq_q));
  const int64_t rows = static_cast<int64_t>(d->batch) * d->heads_q * pad;
  float* dq_acc = static_cast<float*>(workspace);
  float* lse2 = dq_acc + rows * d->d_qk;
  float* delta = lse2 + rows;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);

  CUtensorMap tq, tk, tv, tdo;
  // dO shares O's strides (o_stride); dq/dk/dv share q/k/v strides.
  if (!make_tmap_4d(&tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_qk, d->seq_q, d->heads_q,
                    d->batch, d->q_stride, 64, kBlockM, true) ||
      !make_tmap_4d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_qk, d->seq_k, d->heads_kv,
                    d->batch, d->k_stride, 64, kBlockN, true) ||
      !make_tmap_4d(&tv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_v, d->seq_k, d->heads_kv,
                    d->batch, d->v_stride, 64, kBlockN, true) ||
      !make_tmap_4d(&tdo, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_v, d->seq_q, d->heads_q,
                    d->batch, d->o_stride, 64, kBlockM, true))
    return AF_ERR_INPUT;

  AF_CUDA_CHECK(cudaMemsetAsync(dq_acc, 0, static_cast<size_t>(rows) * d->d_qk * sizeof(float), s));
  {
    const int threads = 256;
    const int64_t warps = rows;
    const unsigned blocks = static_cast<unsigned>((warps * 32 + threads - 1) / threads);
    auto pre = (d->d_v == 128) ? bwd_preprocess_kernel<128> : bwd_preprocess_kernel<64>;
    pre<<<blocks, threads, 0, s>>>(static_cast<const __nv_bfloat16*>(o),
                                   static_cast<const __nv_bfloat16*>(dout), lse, d->o_stride[0],
                                   d->o_stride[1], d->o_stride[2], d->o_stride[0], d->o_stride[1],
                                   d->o_stride[2], d->heads_q, d->seq_q, pad, d->family, lse2,
                                   delta, rows);
    AF_CUDA_CHECK(cudaGetLastError());
  }
  ParallelBwdParams p{};
  p.batch = d->batch; p.heads_q = d->heads_q; p.heads_kv = d->heads_kv;
  p.seq_q = d->seq_q; p.seq_k = d->seq_k; p.d_qk = d->d_qk; p.d_v = d->d_v;
  p.scale = d->scale; p.scale_log2 = d->scale * kLog2e;
  p.mask.causal = d->causal; p.mask.diag_offset = d->diag_offset; p.mask.window = d->window;
  p.act = d->act; p.slope = d->slope; p.bias = d->bias;
  p.lse = lse2; p.delta = delta; p.dq_accum = dq_acc;
  p.dk = dk; p.dv = dv;
  p.dk_stride_b = d->k_stride[0]; p.dk_stride_h = d->k_stride[1]; p.dk_stride_s = d->k_stride[2];
  p.dv_stride_b = d->v_stride[0]; p.dv_stride_h = d->v_stride[1]; p.dv_stride_s = d->v_stride[2];
  if (d->d_qk == 128 && d->d_v == 128) st = dispatch_bwd<128, 128>(d, tq, tk, tv, tdo, p, lse2, delta, pad, s);
  else if (d->d_qk == 64 && d->d_v == 64) st = dispatch_bwd<64, 64>(d, tq, tk, tv, tdo, p, lse2, delta, pad, s);
  else {
    set_error("bf16 parallel backward: head dims (%d, %d) not instantiated", d->d_qk, d->d_v);
    return AF_ERR_UNSUPPORTED;
  }
  if (st != AF_OK) return st;
  {
    const int64_t total_rows = static_cast<int64_t>(d->batch) * d->heads_q * d->seq_q;
    const int64_t threads_total = total_rows * (d->d_qk / 8);
    const unsigned blocks = static_cast<unsigned>((threads_total + 255) / 256);
    auto conv = (d->d_qk == 128) ? bwd_dq_convert_kernel<128> : bwd_dq_convert_kernel<64>;
    conv<<<blocks, 256, 0, s>>>(dq_acc, static_cast<__nv_bfloat16*>(dq), d->q_stride[0],
                                d->q_stride[1], d->q_stride[2], d->heads_q, d->seq_q, pad,
                                d->scale, total_rows);
    AF_CUDA_CHECK(cudaGetLastError());
  }
  return AF_OK;
}

#ifdef AF_TRACE
extern "C" int af_debug_trace_read(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, af::g_af_trace, sizeof(af::g_af_trace)));
}
#endif
