// C-ABI entry points of the parallel-template backward: workspace sizing, the row-statistics
// preprocess, then either K2f (fused 5-GEMM kernel, dQ through an fp32 L2 reduce-add and a convert
// pass; the default for 128/128 heads) or K2a (dK, dV) + K2b (dQ) — no atomics, bitwise
// deterministic (AF_BWD_SPLIT, and every other head-dim pair).  Stream-ordered.
#include "host_common.h"
#include "parallel_bwd.cuh"
#include "parallel_bwd_fused.cuh"

namespace af {
int validate_parallel(const af_parallel_desc* d);
size_t mla_bwd_workspace(const af_parallel_desc* d);
bool materialized_bwd_dims(const af_parallel_desc* d);
int mla_bwd(const af_parallel_desc* d, const void* q, const void* k, const void* v, const void* o,
            const float* lse, const void* dout, void* dq, void* dk, void* dv, void* workspace,
            cudaStream_t s);
inline bool is_mla(const af_parallel_desc* d) { return d->d_qk == 576 && d->d_v == 512; }
namespace {

inline int64_t pad_q(int seq_q) { return ((seq_q + kBlockM - 1) / kBlockM) * kBlockM; }

struct BwdLaunch {
  const af_parallel_desc* d;
  CUtensorMap tq, tk, tv, tdo;
  CUtensorMap tq64, tdo64;  // 64-row query boxes (fused kernel)
  CUtensorMap tdk, tdv;     // dK / dV stores (fused kernel): [32 rows][64 cols] boxes
  bool fused;
  float* dq_accum;
  ParallelBwdParams p;
  const void* q;
  const void* dout;
  void* dq;
  const float* lse2;
  const float* delta;
  int pad;
  cudaStream_t s;
};

template <int D, int DV, int kFamily, int kAct>
int launch_bwd(const BwdLaunch& a) {
  if constexpr (D == 128 && DV == 128) {
    if (a.fused) {
      using L = BwdFusedSmem<D, DV>;  // (the dQ accumulator was zeroed by bwd_preprocess)
      auto kern = parallel_bwd_fused_kernel<D, DV, kFamily, kAct>;
      AF_SMEM_ATTR(kern, L::kTotal);
      dim3 grid((a.d->seq_k + kBlockN - 1) / kBlockN, a.d->batch * a.d->heads_kv);
      ::af::note_launch();
      kern<<<grid, kFusedThreads, L::kTotal, a.s>>>(a.tq64, a.tk, a.tv, a.tdo64, a.tdk, a.tdv,
                                                    a.p, a.lse2, a.delta, a.pad, a.dq_accum);
      AF_CUDA_CHECK(cudaGetLastError());
      const int64_t rows = static_cast<int64_t>(a.d->batch) * a.d->heads_q * a.d->seq_q;
      const int64_t threads = rows * (D / 8);
      ::af::note_launch();
      dq_convert_kernel<D><<<static_cast<unsigned>((threads + 255) / 256), 256, 0, a.s>>>(
          a.dq_accum, static_cast<__nv_bfloat16*>(a.dq), a.d->q_stride[0], a.d->q_stride[1],
          a.d->q_stride[2], a.d->heads_q, a.d->seq_q, a.pad, a.d->scale, rows);
      AF_CUDA_CHECK(cudaGetLastError());
      return AF_OK;
    }
  }
  {
    using L = BwdKVSmem<D, DV>;
    auto kern = parallel_bwd_dkdv_kernel<D, DV, kFamily, kAct>;
    AF_SMEM_ATTR(kern, L::kTotal);
    dim3 grid((a.d->seq_k + kBlockN - 1) / kBlockN, a.d->batch * a.d->heads_kv);
    ::af::note_launch();
    kern<<<grid, kKvThreads, L::kTotal, a.s>>>(a.tq, a.tk, a.tv, a.tdo, a.p, a.lse2, a.delta,
                                               a.pad);
    AF_CUDA_CHECK(cudaGetLastError());
  }
  {
    using L = BwdQSmem<D, DV>;
    auto kern = parallel_bwd_dq_kernel<D, DV, kFamily, kAct>;
    AF_SMEM_ATTR(kern, L::kTotal);
    dim3 grid((a.d->seq_q + kBlockM - 1) / kBlockM, a.d->batch * a.d->heads_q);
    ::af::note_launch();
    kern<<<grid, kDqThreads, L::kTotal, a.s>>>(
        a.tk, a.tv, a.p, static_cast<const __nv_bfloat16*>(a.q),
        static_cast<const __nv_bfloat16*>(a.dout), a.d->q_stride[0], a.d->q_stride[1],
        a.d->q_stride[2], a.d->o_stride[0], a.d->o_stride[1], a.d->o_stride[2], a.dq, a.lse2,
        a.delta, a.pad);
    AF_CUDA_CHECK(cudaGetLastError());
  }
  return AF_OK;
}

template <int D, int DV>
int dispatch_bwd(const BwdLaunch& a) {
  if (a.d->family == AF_FAMILY_SOFTMAX) {
    if (a.d->cap_b != 0.0f) return launch_bwd<D, DV, kFamilySoftmax, kActSoftcap>(a);
    return launch_bwd<D, DV, kFamilySoftmax, kActIdentity>(a);
  }
  if (a.d->family == AF_FAMILY_ABSSUM) return launch_bwd<D, DV, kFamilyAbssum, kActIdentity>(a);
  switch (a.d->act) {
    case AF_ACT_SIGMOID: return launch_bwd<D, DV, kFamilyElementwise, kActSigmoid>(a);
    case AF_ACT_RELU: return launch_bwd<D, DV, kFamilyElementwise, kActRelu>(a);
    case AF_ACT_RELU2: return launch_bwd<D, DV, kFamilyElementwise, kActRelu2>(a);
    case AF_ACT_IDENTITY: return launch_bwd<D, DV, kFamilyElementwise, kActIdentity>(a);
    default: break;
  }
  set_error("unknown activation %d", a.d->act);
  return AF_ERR_INPUT;
}

}  // namespace
}  // namespace af

namespace af {
namespace {
// The 5-GEMM kernel serves the 128/128 head dims unless the split (bitwise-deterministic) pair is
// requested.
bool use_fused_bwd(const af_parallel_desc* d) {
  return d->d_qk == 128 && d->d_v == 128 && d->dtype == AF_DTYPE_BF16 && !is_mla(d) &&
         d->bwd_mode != AF_BWD_SPLIT;
}
}  // namespace
}  // namespace af

extern "C" size_t af_parallel_bwd_workspace(const af_parallel_desc* d) {
  if (d == nullptr) return 0;
  if (af::materialized_bwd_dims(d)) return af::mla_bwd_workspace(d);
  const int64_t rows = static_cast<int64_t>(d->batch) * d->heads_q * af::pad_q(d->seq_q);
  size_t bytes = static_cast<size_t>(rows) * 2 * sizeof(float);
  if (af::use_fused_bwd(d)) bytes += static_cast<size_t>(rows) * d->d_qk * sizeof(float);
  return bytes;
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
  AF_REQUIRE((d->family != AF_FAMILY_SOFTMAX && d->family != AF_FAMILY_ABSSUM) || lse != nullptr,
             AF_ERR_INPUT, "softmax / abssum backward needs the forward row statistic (lse)");
  AF_REQUIRE(d->q_stride[3] == 1 && d->o_stride[3] == 1, AF_ERR_INPUT, "feature stride must be 1");
  if (is_mla(d)) {
    // MLA lowering: V = K[:, :512] of one latent head; dk receives dK + [dV, 0], dv is unused
    AF_REQUIRE(v == k && d->cap_b == 0.0f && d->v_stride[0] == d->k_stride[0] &&
                   d->v_stride[2] == d->k_stride[2],
               AF_ERR_UNSUPPORTED, "(576, 512) heads are lowered only as MLA (V = K[:, :512])");
    return mla_bwd(d, q, k, v, o, lse, dout, dq, dk, dv, workspace,
                   reinterpret_cast<cudaStream_t>(stream));
  }
  if (materialized_bwd_dims(d))  // head dims beyond K2's TMEM budget: (192, 128), (128, 256)
    return mla_bwd(d, q, k, v, o, lse, dout, dq, dk, dv, workspace,
                   reinterpret_cast<cudaStream_t>(stream));
  if (!((d->d_qk == 128 && d->d_v == 128) || (d->d_qk == 64 && d->d_v == 64))) {
    set_error("bf16 parallel backward: head dims (%d, %d) not instantiated", d->d_qk, d->d_v);
    return AF_ERR_UNSUPPORTED;
  }
  BwdLaunch a{};
  a.d = d;
  a.pad = static_cast<int>(pad_q(d->seq_q));
  const int64_t rows = static_cast<int64_t>(d->batch) * d->heads_q * a.pad;
  float* lse2 = static_cast<float*>(workspace);
  float* delta = lse2 + rows;
  a.lse2 = lse2;
  a.delta = delta;
  a.fused = use_fused_bwd(d);
  a.dq_accum = a.fused ? delta + rows : nullptr;
  a.q = q;
  a.dout = dout;
  a.dq = dq;
  a.s = reinterpret_cast<cudaStream_t>(stream);

  // dO shares O's strides (o_stride); dq/dk/dv share q/k/v strides.
  if (!make_tmap_4d(&a.tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_qk, d->seq_q, d->heads_q,
                    d->batch, d->q_stride, 64, kBlockM, true) ||
      !make_tmap_4d(&a.tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_qk, d->seq_k, d->heads_kv,
                    d->batch, d->k_stride, 64, kBlockN, true) ||
      !make_tmap_4d(&a.tv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_v, d->seq_k, d->heads_kv,
                    d->batch, d->v_stride, 64, kBlockN, true) ||
      !make_tmap_4d(&a.tdo, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_v, d->seq_q,
                    d->heads_q, d->batch, d->o_stride, 64, kBlockM, true))
    return AF_ERR_INPUT;
  if (a.fused &&
      (!make_tmap_4d(&a.tq64, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_qk, d->seq_q,
                     d->heads_q, d->batch, d->q_stride, 64, kFusedBM, true) ||
       !make_tmap_4d(&a.tdo64, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_v, d->seq_q,
                     d->heads_q, d->batch, d->o_stride, 64, kFusedBM, true)))
    return AF_ERR_INPUT;

  {
    const int threads = 256;
    const int tpr = d->d_v == 128 ? 4 : 2;  // threads per row (DV / 32)
    const unsigned blocks = static_cast<unsigned>((rows * tpr + threads - 1) / threads);
    auto pre = (d->d_v == 128) ? bwd_preprocess_kernel<128> : bwd_preprocess_kernel<64>;
    ::af::note_launch();
    pre<<<blocks, threads, 0, a.s>>>(static_cast<const __nv_bfloat16*>(o),
                                     static_cast<const __nv_bfloat16*>(dout), lse, d->o_stride[0],
                                     d->o_stride[1], d->o_stride[2], d->o_stride[0],
                                     d->o_stride[1], d->o_stride[2], d->heads_q, d->seq_q, a.pad,
                                     (d->family == AF_FAMILY_ABSSUM && d->cap_a == 0.0f)
                                         ? 3 : d->family,
                                     lse2, delta, rows, a.fused ? a.dq_accum : nullptr);
    AF_CUDA_CHECK(cudaGetLastError());
  }
  ParallelBwdParams& p = a.p;
  p.dkv_tma = (a.fused && d->k_stride[3] == 1 && d->v_stride[3] == 1 &&
               make_tmap_4d(&a.tdk, dk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_qk, d->seq_k,
                            d->heads_kv, d->batch, d->k_stride, 64, 32, true) &&
               make_tmap_4d(&a.tdv, dv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_v, d->seq_k,
                            d->heads_kv, d->batch, d->v_stride, 64, 32, true))
                  ? 1 : 0;
  p.batch = d->batch; p.heads_q = d->heads_q; p.heads_kv = d->heads_kv;
  p.seq_q = d->seq_q; p.seq_k = d->seq_k; p.d_qk = d->d_qk; p.d_v = d->d_v;
  p.scale = d->scale; p.scale_log2 = d->scale * kLog2e;
  p.mask.causal = d->causal; p.mask.diag_offset = d->diag_offset; p.mask.window = d->window;
  p.act = d->act; p.slope = d->slope; p.bias = d->bias;
  p.cap_a = d->cap_a; p.cap_b = d->cap_b;
  p.lse = lse2; p.delta = delta; p.dq_accum = nullptr;
  p.dk = dk; p.dv = dv;
  p.dk_stride_b = d->k_stride[0]; p.dk_stride_h = d->k_stride[1]; p.dk_stride_s = d->k_stride[2];
  p.dv_stride_b = d->v_stride[0]; p.dv_stride_h = d->v_stride[1]; p.dv_stride_s = d->v_stride[2];
  if (d->d_qk == 128) return dispatch_bwd<128, 128>(a);
  return dispatch_bwd<64, 64>(a);
}

#ifdef AF_FUSED_TRACE
extern "C" int af_debug_fused_trace(void* host) {
  return static_cast<int>(
      cudaMemcpyFromSymbol(host, af::g_fused_trace, sizeof(af::g_fused_trace)));
}
#endif
#ifdef AF_BWD_TRACE
extern "C" int af_debug_bwd_trace(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, af::g_bwd_trace, sizeof(af::g_bwd_trace)));
}
extern "C" int af_debug_bwd2a_trace(void* host) {
  return static_cast<int>(
      cudaMemcpyFromSymbol(host, af::g_bwd2a_trace, sizeof(af::g_bwd2a_trace)));
}
#endif
