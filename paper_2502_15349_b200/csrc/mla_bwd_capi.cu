// Host side of K3b, the materialised softmax backward (mla_bwd.cuh): workspace layout, tensor maps
// and the launches (row statistics, scores, dQ GEMM(s), key-side GEMM(s), group reduces).  Called
// by af_parallel_bwd for the MLA lowering ((Dqk, Dv) = (576, 512), one KV head, V = K[:, :512])
// and for the head-dim pairs K2 cannot hold in TMEM: (192, 128) and (128, 256).
#include <algorithm>

#include "host_common.h"
#include "mla_bwd.cuh"
#include "parallel_bwd.cuh"

namespace af {
namespace {

// query / key tiles come in pairs (the CTA-pair kernels): both axes padded to 256
constexpr int64_t pad256(int64_t x) { return ((x + 255) / 256) * 256; }

struct MatLayout {
  int64_t q_pad, k_pad, rows, groups, part_width;
  size_t stats, scores, part, total;
};

MatLayout mat_layout(const af_parallel_desc* d, bool shared) {
  MatLayout l{};
  l.q_pad = pad256(d->seq_q);
  l.k_pad = pad256(d->seq_k);
  l.rows = static_cast<int64_t>(d->batch) * d->heads_q * l.q_pad;
  // head chunks of the key-side GEMMs: enough CTAs for ~4 waves, at most one chunk per head
  const int64_t k_tiles = l.k_pad / 128;
  const int64_t units = k_tiles * d->batch * d->heads_kv;
  const int64_t group = d->heads_q / d->heads_kv;
  const int64_t want =
      d->head_groups > 0 ? d->head_groups : (4 * sm_count() + units - 1) / units;
  l.groups = std::max<int64_t>(1, std::min<int64_t>(want, group));
  l.part_width = shared ? d->d_qk : std::max(d->d_qk, d->d_v);
  l.stats = static_cast<size_t>(l.rows) * 2 * sizeof(float);
  l.scores = static_cast<size_t>(l.rows) * l.k_pad * 2;  // one bf16 [B*H, q_pad, k_pad] buffer
  l.part = static_cast<size_t>(l.groups) * d->batch * d->heads_kv * l.k_pad * l.part_width *
           sizeof(float);
  l.total = l.stats + 2 * l.scores + l.part;
  return l;
}

// 3-D bf16 tensor map [outer][rows][cols] (cols contiguous) as a 4-D map with a unit batch.
bool tmap_3d(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t outer,
             int box_cols, int box_rows) {
  const int64_t st[4] = {0, rows * cols, cols, 1};
  return make_tmap_4d(m, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, static_cast<int>(cols),
                      static_cast<int>(rows), static_cast<int>(outer), 1, st, box_cols, box_rows,
                      true);
}

// N a multiple of 128: the CTA-pair GEMM (each CTA streams half of B); else one CTA per tile
template <int kMode, int N>
int launch_gemm(const CUtensorMap& a1, const CUtensorMap& a2, const CUtensorMap& b1,
                const CUtensorMap& b2, const MlaBwdParams& p, int n0, unsigned grid,
                cudaStream_t s, const CUtensorMap* out = nullptr) {
  ::af::note_launch();
  if constexpr (N % 128 == 0) {
    auto kern = mla_bwd_gemm_pair_kernel<kMode, N>;
    AF_SMEM_ATTR(kern, MlaPairGemmSmem<N>::kTotal);
    MlaBwdParams q = p;
    q.dq_tma = (kMode == kGemmDQ && out != nullptr) ? p.dq_tma : 0;
    q.part_tma = (kMode != kGemmDQ && out != nullptr && N == 512) ? p.part_tma : 0;
    kern<<<grid, 192, MlaPairGemmSmem<N>::kTotal, s>>>(a1, a2, b1, b2, out != nullptr ? *out : a1,
                                                       q, n0);
  } else {
    auto kern = mla_bwd_gemm_kernel<kMode, N>;
    AF_SMEM_ATTR(kern, MlaGemmSmem<N>::kTotal);
    kern<<<grid, 192, MlaGemmSmem<N>::kTotal, s>>>(a1, a2, b1, b2, p, n0);
  }
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

int launch_reduce(const MlaBwdParams& p, const MatLayout& l, const af_parallel_desc* d,
                  int width, void* out, const int64_t* out_stride, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(d->batch) * d->heads_kv * d->seq_k * (width / 4);
  ::af::note_launch();
  mla_bwd_reduce_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
      p.dkv_part, static_cast<int>(l.groups), d->batch * d->heads_kv, d->heads_kv, d->seq_k,
      static_cast<int>(l.k_pad), width, static_cast<int>(l.part_width),
      static_cast<__nv_bfloat16*>(out), out_stride[0],
      out_stride[1], out_stride[2]);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

template <int D, int DV, bool kShared>
int run_materialized(const af_parallel_desc* d, const void* q, const void* k, const void* v,
                     const void* o, const float* lse, const void* dout, void* dq, void* dk,
                     void* dv, void* workspace, cudaStream_t s) {
  const MatLayout l = mat_layout(d, kShared);
  float* lse2 = static_cast<float*>(workspace);
  float* delta = lse2 + l.rows;
  uint8_t* base = static_cast<uint8_t*>(workspace) + l.stats;
  auto* pbuf = reinterpret_cast<__nv_bfloat16*>(base);
  auto* dsbuf = reinterpret_cast<__nv_bfloat16*>(base + l.scores);
  auto* part = reinterpret_cast<float*>(base + 2 * l.scores);

  {  // row statistics: LSE*log2e (+inf when fully masked / padded), D = rowsum(dO*O)
    const int threads = 256;
    const unsigned blocks = static_cast<unsigned>((l.rows * (DV / 32) + threads - 1) / threads);
    ::af::note_launch();
    bwd_preprocess_kernel<DV><<<blocks, threads, 0, s>>>(
        static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), lse,
        d->o_stride[0], d->o_stride[1], d->o_stride[2], d->o_stride[0], d->o_stride[1],
        d->o_stride[2], d->heads_q, d->seq_q, static_cast<int>(l.q_pad), AF_FAMILY_SOFTMAX,
        lse2, delta, l.rows);
    AF_CUDA_CHECK(cudaGetLastError());
  }

  MlaBwdParams p{};
  p.batch = d->batch;
  p.heads = d->heads_q;
  p.heads_kv = d->heads_kv;
  p.seq_q = d->seq_q;
  p.seq_k = d->seq_k;
  p.q_pad = static_cast<int>(l.q_pad);
  p.k_pad = static_cast<int>(l.k_pad);
  p.scale = d->scale;
  p.scale_log2 = d->scale * kLog2e;
  p.mask.causal = d->causal;
  p.mask.diag_offset = d->diag_offset;
  p.mask.window = 0;
  p.lse2 = lse2;
  p.delta = delta;
  p.p = pbuf;
  p.ds = dsbuf;
  p.dq = dq;
  p.dq_sb = d->q_stride[0];
  p.dq_sh = d->q_stride[1];
  p.dq_ss = d->q_stride[2];
  p.dkv_part = part;
  p.groups = static_cast<int>(l.groups);
  p.part_width = static_cast<int>(l.part_width);

  const int64_t bhs = static_cast<int64_t>(d->batch) * d->heads_q;
  const int q_tiles = static_cast<int>(l.q_pad / 128), k_tiles = static_cast<int>(l.k_pad / 128);

  {  // 1. scores: P and dS' = tau P (dP - D) for the visible blocks
    using SL = MlaScoresSmem<D, DV, kShared>;
    CUtensorMap tq, tdo, tk, tv;
    // Q / dO in half boxes: each CTA of a pair streams 64 of a tile's 128 query rows
    if (!make_tmap_4d(&tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, d->seq_q, d->heads_q,
                      d->batch, d->q_stride, 64, 64, true) ||
        !make_tmap_4d(&tdo, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, DV, d->seq_q, d->heads_q,
                      d->batch, d->o_stride, 64, 64, true) ||
        !make_tmap_4d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, d->seq_k, d->heads_kv,
                      d->batch, d->k_stride, 64, 128, true) ||
        !make_tmap_4d(&tv, kShared ? k : v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                      kShared ? D : DV, d->seq_k, d->heads_kv, d->batch,
                      kShared ? d->k_stride : d->v_stride, 64, 128, true))
      return AF_ERR_INPUT;
    CUtensorMap tpst, tdsst;  // P^T / dS'^T stores: [32 key rows][64 query columns] boxes
    if (!tmap_3d(&tpst, pbuf, l.q_pad, l.k_pad, bhs, 64, 32) ||
        !tmap_3d(&tdsst, dsbuf, l.q_pad, l.k_pad, bhs, 64, 32))
      return AF_ERR_INPUT;
    auto kern = mla_bwd_scores_kernel<D, DV, kShared>;
    AF_SMEM_ATTR(kern, SL::kTotal);
    ::af::note_launch();
    kern<<<static_cast<unsigned>(k_tiles * bhs), 320, SL::kTotal, s>>>(tq, tdo, tk, tv, tpst,
                                                                         tdsst, p);
    AF_CUDA_CHECK(cudaGetLastError());
  }

  // maps shared by the GEMMs
  CUtensorMap tds_q, tds_k, tp_k, tkb, tqb, tdob;
  // P^T / dS'^T are [b*H, k_pad, q_pad]: the dQ GEMM reads [64 keys][64 queries] boxes
  // (MN-major A), the key-side GEMMs [128 keys][64 queries] boxes (K-major A)
  if (!tmap_3d(&tds_q, dsbuf, l.q_pad, l.k_pad, bhs, 64, 64) ||
      !tmap_3d(&tds_k, dsbuf, l.q_pad, l.k_pad, bhs, 64, 128) ||
      !tmap_3d(&tp_k, pbuf, l.q_pad, l.k_pad, bhs, 64, 128) ||
      !make_tmap_4d(&tkb, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, d->seq_k, d->heads_kv,
                    d->batch, d->k_stride, 64, 64, true) ||
      !make_tmap_4d(&tqb, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, d->seq_q, d->heads_q,
                    d->batch, d->q_stride, 64, 64, true) ||
      !make_tmap_4d(&tdob, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, DV, d->seq_q, d->heads_q,
                    d->batch, d->o_stride, 64, 64, true))
    return AF_ERR_INPUT;
  const unsigned gq = static_cast<unsigned>(q_tiles * bhs);
  const unsigned gk = static_cast<unsigned>(k_tiles * d->batch * d->heads_kv * l.groups);
  int st;
  // dQ leaves the pair GEMM through TMA stores of [32 rows][64 cols] boxes when it can be mapped
  CUtensorMap tdq;
  p.dq_tma = (d->q_stride[3] == 1 &&
              make_tmap_4d(&tdq, dq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, d->seq_q,
                           d->heads_q, d->batch, d->q_stride, 64, 32, true))
                 ? 1 : 0;
  // the key-side partials [G, B*Hkv, k_pad, width] fp32 through [32 rows][32 cols] boxes
  CUtensorMap tpart;
  const int64_t part_st[4] = {static_cast<int64_t>(d->batch) * d->heads_kv * l.k_pad * l.part_width,
                              l.k_pad * l.part_width, l.part_width, 1};
  p.part_tma = make_tmap_4d(&tpart, part, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                            static_cast<int>(l.part_width), static_cast<int>(l.k_pad),
                            d->batch * d->heads_kv, static_cast<int>(l.groups), part_st, 32, 32,
                            true)
                   ? 1 : 0;
#ifdef AF_MLA_PART_ROWSTORES  // developer ablation: per-thread row stores of the partials
  p.part_tma = 0;
#endif
  if constexpr (kShared) {  // MLA: dQ in 512 + 64 columns, one latent dKV accumulator
    if ((st = launch_gemm<kGemmDQ, 512>(tds_q, tds_q, tkb, tkb, p, 0, gq, s, &tdq)) != AF_OK)
      return st;
    if ((st = launch_gemm<kGemmDQ, 64>(tds_q, tds_q, tkb, tkb, p, 512, gq, s)) != AF_OK) return st;
    if ((st = launch_gemm<kGemmDKV, 512>(tds_k, tp_k, tqb, tdob, p, 0, gk, s, &tpart)) != AF_OK)
      return st;
    if ((st = launch_gemm<kGemmDKV, 64>(tds_k, tp_k, tqb, tdob, p, 512, gk, s)) != AF_OK) return st;
    return launch_reduce(p, l, d, D, dk, d->k_stride, s);
  } else {
    if ((st = launch_gemm<kGemmDQ, D>(tds_q, tds_q, tkb, tkb, p, 0, gq, s, &tdq)) != AF_OK)
      return st;
    if ((st = launch_gemm<kGemmDK, D>(tds_k, tp_k, tqb, tdob, p, 0, gk, s)) != AF_OK) return st;
    if ((st = launch_reduce(p, l, d, D, dk, d->k_stride, s)) != AF_OK) return st;
    if ((st = launch_gemm<kGemmDV, DV>(tds_k, tp_k, tqb, tdob, p, 0, gk, s)) != AF_OK) return st;
    return launch_reduce(p, l, d, DV, dv, d->v_stride, s);
  }
}

}  // namespace

bool materialized_bwd_dims(const af_parallel_desc* d) {
  return (d->d_qk == 576 && d->d_v == 512) || (d->d_qk == 192 && d->d_v == 128) ||
         (d->d_qk == 128 && d->d_v == 256);
}

// The materialised path holds two bf16 [b*H, q_pad, k_pad] score buffers: it runs over chunks
// of the batch whose workspace fits kMatBudget, so the scratch stays bounded at any batch size
// (e.g. softmax-diff 128/256 at B8 H32 S8192 would need ~68 GB in one pass).  A single batch
// element above the budget is unsupported.
constexpr size_t kMatBudget = size_t(24) << 30;

int mat_batch_chunk(const af_parallel_desc* d) {
  af_parallel_desc c = *d;
  const bool shared = d->d_qk == 576 && d->d_v == 512;
  int lo = 1;
  for (int b = d->batch; b >= 1; b = (b == 1 ? 0 : (b + 1) / 2)) {
    c.batch = b;
    if (mat_layout(&c, shared).total <= kMatBudget) {
      lo = b;
      break;
    }
    if (b == 1) return 0;
  }
  return lo;
}

size_t mla_bwd_workspace(const af_parallel_desc* d) {
  const int chunk = mat_batch_chunk(d);
  af_parallel_desc c = *d;
  c.batch = chunk > 0 ? chunk : 1;
  return mat_layout(&c, d->d_qk == 576 && d->d_v == 512).total;
}

int mla_bwd(const af_parallel_desc* d, const void* q, const void* k, const void* v, const void* o,
            const float* lse, const void* dout, void* dq, void* dk, void* dv, void* workspace,
            cudaStream_t s) {
  AF_REQUIRE(d->family == AF_FAMILY_SOFTMAX && d->cap_b == 0.0f, AF_ERR_UNSUPPORTED,
             "the materialised backward (head dims %d/%d) is softmax only", d->d_qk, d->d_v);
  AF_REQUIRE(!d->causal || d->diag_offset == 0, AF_ERR_UNSUPPORTED,
             "the materialised backward supports the top-left causal mask (offset 0) only");
  AF_REQUIRE(d->window <= 0, AF_ERR_UNSUPPORTED, "the materialised backward has no sliding window");
  AF_REQUIRE(d->k_stride[3] == 1 && d->q_stride[3] == 1 && d->o_stride[3] == 1 &&
                 d->v_stride[3] == 1,
             AF_ERR_INPUT, "feature stride must be 1");
  const int chunk = mat_batch_chunk(d);
  AF_REQUIRE(chunk > 0, AF_ERR_UNSUPPORTED,
             "materialised backward: one batch element needs more than %zu GB of score scratch "
             "(heads %d, seq %d x %d)", kMatBudget >> 30, d->heads_q, d->seq_q, d->seq_k);
  auto off = [](const void* p, int64_t elems, int bytes) {
    return p == nullptr ? nullptr
                        : static_cast<const void*>(static_cast<const char*>(p) + elems * bytes);
  };
  for (int b0 = 0; b0 < d->batch; b0 += chunk) {
    af_parallel_desc c = *d;
    c.batch = std::min(chunk, d->batch - b0);
    const void* q_ = off(q, b0 * d->q_stride[0], 2);
    const void* k_ = off(k, b0 * d->k_stride[0], 2);
    const void* v_ = off(v, b0 * d->v_stride[0], 2);
    const void* o_ = off(o, b0 * d->o_stride[0], 2);
    const void* do_ = off(dout, b0 * d->o_stride[0], 2);
    const float* lse_ = static_cast<const float*>(
        off(lse, static_cast<int64_t>(b0) * d->heads_q * d->seq_q, 4));
    void* dq_ = const_cast<void*>(off(dq, b0 * d->q_stride[0], 2));
    void* dk_ = const_cast<void*>(off(dk, b0 * d->k_stride[0], 2));
    void* dv_ = const_cast<void*>(off(dv, b0 * d->v_stride[0], 2));
    int st = AF_ERR_UNSUPPORTED;
    if (d->d_qk == 576 && d->d_v == 512) {
      AF_REQUIRE(d->heads_kv == 1, AF_ERR_UNSUPPORTED, "MLA backward needs one latent KV head");
      st = run_materialized<576, 512, true>(&c, q_, k_, v_, o_, lse_, do_, dq_, dk_, dv_,
                                            workspace, s);
    } else if (d->d_qk == 192 && d->d_v == 128) {
      st = run_materialized<192, 128, false>(&c, q_, k_, v_, o_, lse_, do_, dq_, dk_, dv_,
                                             workspace, s);
    } else if (d->d_qk == 128 && d->d_v == 256) {
      st = run_materialized<128, 256, false>(&c, q_, k_, v_, o_, lse_, do_, dq_, dk_, dv_,
                                             workspace, s);
    } else {
      set_error("materialised backward: head dims (%d, %d) not instantiated", d->d_qk, d->d_v);
      return AF_ERR_UNSUPPORTED;
    }
    if (st != AF_OK) return st;
  }
  return AF_OK;
}

}  // namespace af

#ifdef AF_SCORES_TRACE
extern "C" int af_debug_scores_trace(void* host, int reset) {
  if (reset) {
    static long long zero[256][8];
    return static_cast<int>(cudaMemcpyToSymbol(af::g_scores_trace, zero, sizeof(zero)));
  }
  return static_cast<int>(cudaMemcpyFromSymbol(host, af::g_scores_trace,
                                               sizeof(af::g_scores_trace)));
}
#endif
