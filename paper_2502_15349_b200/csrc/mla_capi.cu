// C-ABI for K3 (MLA): decode entry point + the prefill launcher used by af_parallel_fwd when the
// variant is softmax over one shared latent head with (Dqk, Dv) = (576, 512) and V = K[:, :512].
#include "host_common.h"
#include "mla.cuh"

namespace af {

using PrefillSmem = MlaSmem<MlaTile<false>::kN, MlaTile<false>::kStages, MlaTile<false>::kQT>;
using DecodeSmem = MlaSmem<MlaTile<true>::kN, MlaTile<true>::kStages, MlaTile<true>::kQT>;

int mla_prefill(const af_parallel_desc* d, const void* q, const void* k, void* o, float* lse,
                cudaStream_t s) {
  AF_REQUIRE(d->heads_kv == 1, AF_ERR_UNSUPPORTED, "MLA prefill needs one latent KV head");
  CUtensorMap tq, tkv;
  const int64_t kv_st[4] = {0, d->k_stride[0], d->k_stride[2], 1};  // dims (576, Sk, B, 1)
  if (!make_tmap_4d(&tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMlaDqk, d->seq_q, d->heads_q,
                    d->batch, d->q_stride, 64, 128, true) ||
      !make_tmap_4d(&tkv, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMlaDqk, d->seq_k, d->batch, 1,
                    kv_st, 64, MlaTile<false>::kN, true))
    return AF_ERR_INPUT;
  MlaParams p{};
  p.batch = d->batch; p.heads = d->heads_q; p.seq_q = d->seq_q; p.seq_k = d->seq_k;
  p.scale_log2 = d->scale * kLog2e;
  AF_REQUIRE(!d->causal || d->diag_offset == 0, AF_ERR_UNSUPPORTED,
             "MLA prefill supports the top-left causal mask (offset 0) only");
  AF_REQUIRE(d->window <= 0, AF_ERR_UNSUPPORTED, "MLA prefill has no sliding window");
  p.causal = d->causal;
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.q_sb = d->q_stride[0]; p.q_sh = d->q_stride[1]; p.q_ss = d->q_stride[2];
  p.o = o; p.o_sb = d->o_stride[0]; p.o_sh = d->o_stride[1]; p.o_ss = d->o_stride[2];
  p.lse = lse;
  CUtensorMap to{};
  p.o_tma = (d->o_stride[3] == 1 &&
             make_tmap_4d(&to, o, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMlaDv, d->seq_q,
                          d->heads_q, d->batch, d->o_stride, 64, 32, true))
                ? 1 : 0;
  auto kern = mla_fwd_kernel<false>;
  AF_SMEM_ATTR(kern, PrefillSmem::kTotal);
  const int q_tiles = (d->seq_q + 127) / 128;
  ::af::note_launch();
  kern<<<q_tiles * d->batch * d->heads_q * 2, 192, PrefillSmem::kTotal, s>>>(tq, tkv, to, p);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

namespace {
// KV splits per (batch, value half): one CTA per SM (TMEM / smem), so the step time is
// waves x blocks-per-CTA; pick the split count minimising it (plus a fixed per-CTA cost of
// ~4 key blocks for the Q load, pipeline fill and partial-O write), e.g. B=16 on 148 SMs gives
// 9 splits = 288 CTAs in two waves rather than 10 = 320 CTAs in three.
int decode_splits(const af_mla_desc* d) {
  const int sms = sm_count();
  const int blocks = (d->seq_k + MlaTile<true>::kN - 1) / MlaTile<true>::kN;
  if (d->splits > 0) return std::min(d->splits, blocks);  // the measured scheduler's choice
  const int max_splits = std::max(1, std::min(blocks, 8 * sms / (2 * d->batch) + 1));
  int best = 1;
  long best_cost = -1;
  for (int s = 1; s <= max_splits; ++s) {
    const long ctas = 2L * d->batch * s;
    const long waves = (ctas + sms - 1) / sms;
    const long cost = waves * ((blocks + s - 1) / s + 4);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}
}  // namespace

}  // namespace af

extern "C" size_t af_mla_decode_workspace(const af_mla_desc* d) {
  if (d == nullptr) return 0;
  const size_t rows = static_cast<size_t>(d->batch) * af::decode_splits(d) * d->heads;
  return rows * (af::kMlaDv + 1) * sizeof(float);
}

extern "C" int af_mla_decode(const af_mla_desc* d, const void* q, const void* kv, void* o,
                             float* lse, void* workspace, size_t workspace_bytes, void* stream) {
  using namespace af;
  AF_REQUIRE(d != nullptr, AF_ERR_INPUT, "null descriptor");
  AF_REQUIRE(d->d_qk == kMlaDqk && d->d_v == kMlaDv, AF_ERR_UNSUPPORTED,
             "MLA decode is built for (Dqk, Dv) = (576, 512), got (%d, %d)", d->d_qk, d->d_v);
  AF_REQUIRE(d->heads >= 1 && d->heads <= 128, AF_ERR_UNSUPPORTED,
             "MLA decode packs the heads of one token into a 128-row tile (heads=%d)", d->heads);
  AF_REQUIRE(d->batch >= 1 && d->seq_k >= 1, AF_ERR_INPUT, "dims must be >= 1");
  AF_REQUIRE(workspace_bytes >= af_mla_decode_workspace(d), AF_ERR_INPUT, "workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int splits = decode_splits(d);
  int split_len = (d->seq_k + splits - 1) / splits;
  split_len = ((split_len + MlaTile<true>::kN - 1) / MlaTile<true>::kN) * MlaTile<true>::kN;
  // q [B, H, 576] and kv [B, Sk, 576], contiguous
  CUtensorMap tq, tkv;
  const int64_t q_st[4] = {0, static_cast<int64_t>(d->heads) * kMlaDqk, kMlaDqk, 1};  // (576, H, B, 1)
  const int64_t kv_st[4] = {0, static_cast<int64_t>(d->seq_k) * kMlaDqk, kMlaDqk, 1};
  if (!make_tmap_4d(&tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMlaDqk, d->heads, d->batch, 1,
                    q_st, 64, 128, true) ||
      !make_tmap_4d(&tkv, kv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMlaDqk, d->seq_k, d->batch, 1,
                    kv_st, 64, MlaTile<true>::kN, true))
    return AF_ERR_INPUT;
  MlaParams p{};
  p.batch = d->batch; p.heads = d->heads; p.seq_q = 1; p.seq_k = d->seq_k;
  p.scale_log2 = d->scale * kLog2e;
  p.causal = 0;
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.q_sb = static_cast<int64_t>(d->heads) * kMlaDqk; p.q_sh = 0; p.q_ss = kMlaDqk;
  p.splits = splits;
  p.split_len = split_len;
  float* part_o = static_cast<float*>(workspace);
  float* part_lse = part_o + static_cast<size_t>(d->batch) * splits * d->heads * kMlaDv;
  p.part_o = part_o;
  p.part_lse = part_lse;
  {
    auto kern = mla_fwd_kernel<true>;
    AF_SMEM_ATTR(kern, DecodeSmem::kTotal);
    ::af::note_launch();
    // partial O [B, splits, H, 512] fp32 as (512, H, splits, B) with [32 heads][32 cols] boxes
    CUtensorMap tpo;
    const int64_t po_st[4] = {static_cast<int64_t>(splits) * d->heads * kMlaDv,
                              static_cast<int64_t>(d->heads) * kMlaDv, kMlaDv, 1};
    p.o_tma = make_tmap_4d(&tpo, part_o, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, kMlaDv, d->heads,
                           splits, d->batch, po_st, 32, 32, true)
                  ? 1 : 0;
    kern<<<d->batch * splits * 2, 192, DecodeSmem::kTotal, s>>>(tq, tkv, p.o_tma ? tpo : tkv, p);
  }
  AF_CUDA_CHECK(cudaGetLastError());
  ::af::note_launch();
  mla_combine_kernel<<<d->batch * d->heads, kMlaDv / 4, 0, s>>>(
      part_o, part_lse, d->batch, d->heads, splits, static_cast<__nv_bfloat16*>(o), lse);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

#ifdef AF_MLA_TRACE
extern "C" int af_debug_mla_trace(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, af::g_mla_trace, sizeof(af::g_mla_trace)));
}
#endif
