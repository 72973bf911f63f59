// C-ABI entry points of the parallel template (forward).  Validates the descriptor, encodes TMA
// tensor maps and dispatches the K1 instantiation for (head dims, hook family, activation).
#include "host_common.h"
#include "parallel_fwd.cuh"

namespace af {
namespace {


template <int D, int DV, int kFamily, int kAct, int kStages>
int launch_fwd_stages(const af_parallel_desc* d, const CUtensorMap& tq, const CUtensorMap& tk,
                      const CUtensorMap& tv, const CUtensorMap& to, const ParallelFwdParams& p,
                      cudaStream_t stream) {
  using L = FwdSmem<D, DV, kStages>;
  auto kern = parallel_fwd_kernel<D, DV, kFamily, kAct, kStages>;
  AF_SMEM_ATTR(kern, L::kTotal);
  dim3 grid((d->seq_q + 2 * kBlockM - 1) / (2 * kBlockM), d->batch * d->heads_q);
  ::af::note_launch();
  kern<<<grid, fwd_threads(kFamily), L::kTotal, stream>>>(tq, tk, tv, to, p);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

template <int D, int DV, int kFamily, int kAct>
int launch_fwd(const af_parallel_desc* d, const CUtensorMap& tq, const CUtensorMap& tk,
               const CUtensorMap& tv, const CUtensorMap& to, const ParallelFwdParams& p,
               cudaStream_t stream) {
  // D = 192: two 48 KB Q tiles leave room for one stage; D <= 128 runs two unless the measured
  // scheduler picked one (desc->kv_stages)
  constexpr bool kTunable = (kFamily == kFamilySoftmax && kAct == kActIdentity) ||
                            (kFamily == kFamilyElementwise && kAct == kActSigmoid);
  if constexpr (D <= 128) {
    if (kTunable && d->kv_stages == 1) return launch_fwd_stages<D, DV, kFamily, kAct, 1>(d, tq, tk, tv, to, p, stream);
    return launch_fwd_stages<D, DV, kFamily, kAct, 2>(d, tq, tk, tv, to, p, stream);
  } else {
    return launch_fwd_stages<D, DV, kFamily, kAct, 1>(d, tq, tk, tv, to, p, stream);
  }
}

template <int D, int DV>
int dispatch_family(const af_parallel_desc* d, const CUtensorMap& tq, const CUtensorMap& tk,
                    const CUtensorMap& tv, const CUtensorMap& to, const ParallelFwdParams& p,
                    cudaStream_t s) {
  if (d->family == AF_FAMILY_SOFTMAX) {
    if (d->cap_b != 0.0f) return launch_fwd<D, DV, kFamilySoftmax, kActSoftcap>(d, tq, tk, tv, to, p, s);
    return launch_fwd<D, DV, kFamilySoftmax, kActIdentity>(d, tq, tk, tv, to, p, s);
  }
  if (d->family == AF_FAMILY_ABSSUM) return launch_fwd<D, DV, kFamilyAbssum, kActIdentity>(d, tq, tk, tv, to, p, s);
  switch (d->act) {
    case AF_ACT_SIGMOID: return launch_fwd<D, DV, kFamilyElementwise, kActSigmoid>(d, tq, tk, tv, to, p, s);
    case AF_ACT_RELU: return launch_fwd<D, DV, kFamilyElementwise, kActRelu>(d, tq, tk, tv, to, p, s);
    case AF_ACT_RELU2: return launch_fwd<D, DV, kFamilyElementwise, kActRelu2>(d, tq, tk, tv, to, p, s);
    case AF_ACT_IDENTITY: return launch_fwd<D, DV, kFamilyElementwise, kActIdentity>(d, tq, tk, tv, to, p, s);
    default: break;
  }
  set_error("unknown activation %d", d->act);
  return AF_ERR_INPUT;
}

}  // namespace

int validate_parallel(const af_parallel_desc* d) {
  AF_REQUIRE(d != nullptr, AF_ERR_INPUT, "null descriptor");
  AF_REQUIRE(d->batch >= 1 && d->heads_q >= 1 && d->heads_kv >= 1 && d->seq_q >= 1 &&
                 d->seq_k >= 1 && d->d_qk >= 1 && d->d_v >= 1,
             AF_ERR_INPUT, "dims must be >= 1");
  AF_REQUIRE(d->heads_q % d->heads_kv == 0, AF_ERR_SHAPE,
             "heads_q (%d) must be a multiple of heads_kv (%d)", d->heads_q, d->heads_kv);
  AF_REQUIRE(d->family == AF_FAMILY_SOFTMAX || d->family == AF_FAMILY_ELEMENTWISE ||
                 d->family == AF_FAMILY_ABSSUM,
             AF_ERR_INPUT, "unknown hook family %d", d->family);
  AF_REQUIRE(d->family != AF_FAMILY_ABSSUM || d->slope != nullptr, AF_ERR_INPUT,
             "abssum family needs the per-head log2 decay (slope)");
  return AF_OK;
}

ParallelFwdParams make_fwd_params(const af_parallel_desc* d, void* o, float* lse) {
  ParallelFwdParams p{};
  p.batch = d->batch;
  p.heads_q = d->heads_q;
  p.heads_kv = d->heads_kv;
  p.seq_q = d->seq_q;
  p.seq_k = d->seq_k;
  p.d_qk = d->d_qk;
  p.d_v = d->d_v;
  p.scale = d->scale;
  p.scale_log2 = d->scale * 1.4426950408889634f;
  p.mask.causal = d->causal;
  p.mask.diag_offset = d->diag_offset;
  p.mask.window = d->window;
  p.act = d->act;
  p.slope = d->slope;
  p.bias = d->bias;
  p.cap_a = d->cap_a;
  p.cap_b = d->cap_b;
  p.o = o;
  p.o_stride_b = d->o_stride[0];
  p.o_stride_h = d->o_stride[1];
  p.o_stride_s = d->o_stride[2];
  p.lse = lse;
  return p;
}

}  // namespace af

namespace af {
int mla_prefill(const af_parallel_desc* d, const void* q, const void* k, void* o, float* lse,
                cudaStream_t s);
}

extern "C" int af_parallel_fwd_f32(const af_parallel_desc* d, const void* q, const void* k,
                                   const void* v, void* o, float* lse, void* stream);

extern "C" int af_parallel_fwd(const af_parallel_desc* d, const void* q, const void* k,
                               const void* v, void* o, float* lse, void* stream) {
  using namespace af;
  int st = validate_parallel(d);
  if (st != AF_OK) return st;
  if (d->dtype == AF_DTYPE_F32) return af_parallel_fwd_f32(d, q, k, v, o, lse, stream);
  AF_REQUIRE(d->dtype == AF_DTYPE_BF16, AF_ERR_INPUT, "unknown dtype %d", d->dtype);
  AF_REQUIRE(d->o_stride[3] == 1, AF_ERR_INPUT, "output feature stride must be 1");
  if (d->d_qk == 576 && d->d_v == 512) {
    // MLA: one latent head, V = K[:, :512] (same base pointer and strides)
    AF_REQUIRE(d->family == AF_FAMILY_SOFTMAX && d->cap_b == 0.0f && v == k &&
                   d->v_stride[0] == d->k_stride[0] &&
                   d->v_stride[2] == d->k_stride[2],
               AF_ERR_UNSUPPORTED, "(576, 512) heads are lowered only as MLA (softmax, V = K[:, :512])");
    return mla_prefill(d, q, k, o, lse, reinterpret_cast<cudaStream_t>(stream));
  }
  CUtensorMap tq, tk, tv;
  if (!make_tmap_4d(&tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_qk, d->seq_q, d->heads_q,
                    d->batch, d->q_stride, 64, kBlockM, true) ||
      !make_tmap_4d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_qk, d->seq_k, d->heads_kv,
                    d->batch, d->k_stride, 64, kBlockN, true) ||
      !make_tmap_4d(&tv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_v, d->seq_k, d->heads_kv,
                    d->batch, d->v_stride, 64, kBlockN, true))
    return AF_ERR_INPUT;
  ParallelFwdParams p = make_fwd_params(d, o, lse);
  // O through TMA stores of staged [32 rows][64 cols] boxes when its strides allow a tensor map
  // (16-byte multiples, feature stride 1); else per-thread row stores
  CUtensorMap to{};
  p.o_tma = (d->o_stride[3] == 1 && d->d_v % 64 == 0 &&
             make_tmap_4d(&to, o, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->d_v, d->seq_q,
                          d->heads_q, d->batch, d->o_stride, 64, 32, true))
                ? 1 : 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (d->d_qk == 128 && d->d_v == 128) return dispatch_family<128, 128>(d, tq, tk, tv, to, p, s);
  if (d->d_qk == 64 && d->d_v == 64) return dispatch_family<64, 64>(d, tq, tk, tv, to, p, s);
  if (d->d_qk == 192 && d->d_v == 128) return dispatch_family<192, 128>(d, tq, tk, tv, to, p, s);
  set_error("bf16 parallel forward: head dims (%d, %d) not instantiated", d->d_qk, d->d_v);
  return AF_ERR_UNSUPPORTED;
}

#ifdef AF_FWD_TRACE
extern "C" int af_debug_fwd_trace(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, af::g_fwd_trace, n * sizeof(unsigned long long)) == cudaSuccess
             ? 0
             : 1;
}
#endif
