// Host side of K3b (MLA backward): workspace layout, tensor maps and the five launches
// (row statistics, scores, dQ GEMM x2, dKV GEMM x2, group reduce).  Called by af_parallel_bwd when
// the descriptor is the MLA lowering ((Dqk, Dv) = (576, 512), one KV head, V = K[:, :512]).
#include "host_common.h"
#include "mla_bwd.cuh"
#include "parallel_bwd.cuh"

namespace af {
namespace {

constexpr int64_t pad128(int64_t x) { return ((x + 127) / 128) * 128; }

struct MlaBwdLayout {
  int64_t q_pad, k_pad, rows, groups;
  size_t stats, scores, part, total;
};

MlaBwdLayout mla_layout(const af_parallel_desc* d) {
  MlaBwdLayout l{};
  l.q_pad = pad128(d->seq_q);
  l.k_pad = pad128(d->seq_k);
  l.rows = static_cast<int64_t>(d->batch) * d->heads_q * l.q_pad;
  // head groups of the dKV GEMM: enough CTAs for ~4 waves, at most one group per head
  const int64_t k_tiles = l.k_pad / 128;
  const int64_t want = (4 * sm_count() + k_tiles * d->batch - 1) / (k_tiles * d->batch);
  l.groups = std::max<int64_t>(1, std::min<int64_t>(want, d->heads_q));
  l.stats = static_cast<size_t>(l.rows) * 2 * sizeof(float);
  l.scores = static_cast<size_t>(l.rows) * l.k_pad * 2;  // one bf16 [B*H, q_pad, k_pad] buffer
  l.part = static_cast<size_t>(l.groups) * d->batch * l.k_pad * kMbDqk * sizeof(float);
  l.total = l.stats + 2 * l.scores + l.part;
  return l;
}

template <typename K>
int set_smem(K kern, int bytes) {
  AF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return AF_OK;
}

// 3-D bf16 tensor map [outer][rows][cols] (cols contiguous) as a 4-D map with a unit batch.
bool tmap_3d(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t outer,
             int box_cols, int box_rows) {
  const int64_t st[4] = {0, rows * cols, cols, 1};
  return make_tmap_4d(m, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, static_cast<int>(cols),
                      static_cast<int>(rows), static_cast<int>(outer), 1, st, box_cols, box_rows,
                      true);
}

}  // namespace

size_t mla_bwd_workspace(const af_parallel_desc* d) { return mla_layout(d).total; }

int mla_bwd(const af_parallel_desc* d, const void* q, const void* k, const void* o,
            const float* lse, const void* dout, void* dq, void* dkv, void* workspace,
            cudaStream_t s) {
  AF_REQUIRE(d->heads_kv == 1, AF_ERR_UNSUPPORTED, "MLA backward needs one latent KV head");
  AF_REQUIRE(d->family == AF_FAMILY_SOFTMAX, AF_ERR_UNSUPPORTED, "MLA backward is softmax only");
  AF_REQUIRE(!d->causal || d->diag_offset == 0, AF_ERR_UNSUPPORTED,
             "MLA backward supports the top-left causal mask (offset 0) only");
  AF_REQUIRE(d->window <= 0, AF_ERR_UNSUPPORTED, "MLA backward has no sliding window");
  AF_REQUIRE(d->k_stride[3] == 1 && d->q_stride[3] == 1 && d->o_stride[3] == 1, AF_ERR_INPUT,
             "feature stride must be 1");
  const MlaBwdLayout l = mla_layout(d);
  float* lse2 = static_cast<float*>(workspace);
  float* delta = lse2 + l.rows;
  uint8_t* base = static_cast<uint8_t*>(workspace) + l.stats;
  auto* pbuf = reinterpret_cast<__nv_bfloat16*>(base);
  auto* dsbuf = reinterpret_cast<__nv_bfloat16*>(base + l.scores);
  auto* part = reinterpret_cast<float*>(base + 2 * l.scores);

  {  // row statistics: LSE*log2e (+inf when fully masked / padded), D = rowsum(dO*O)
    const int threads = 256;
    const unsigned blocks = static_cast<unsigned>((l.rows * 32 + threads - 1) / threads);
    ::af::note_launch();
    bwd_preprocess_kernel<kMbDv><<<blocks, threads, 0, s>>>(
        static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), lse,
        d->o_stride[0], d->o_stride[1], d->o_stride[2], d->o_stride[0], d->o_stride[1],
        d->o_stride[2], d->heads_q, d->seq_q, static_cast<int>(l.q_pad), AF_FAMILY_SOFTMAX,
        lse2, delta, l.rows);
    AF_CUDA_CHECK(cudaGetLastError());
  }

  MlaBwdParams p{};
  p.batch = d->batch;
  p.heads = d->heads_q;
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

  const int64_t kv_st[4] = {0, d->k_stride[0], d->k_stride[2], 1};  // (576, Sk, B, 1)
  const int64_t bhs = static_cast<int64_t>(d->batch) * d->heads_q;
  const int q_tiles = static_cast<int>(l.q_pad / 128), k_tiles = static_cast<int>(l.k_pad / 128);

  {  // 1. scores
    CUtensorMap tq, tdo, tk;
    if (!make_tmap_4d(&tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMbDqk, d->seq_q, d->heads_q,
                      d->batch, d->q_stride, 64, 128, true) ||
        !make_tmap_4d(&tdo, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMbDv, d->seq_q,
                      d->heads_q, d->batch, d->o_stride, 64, 128, true) ||
        !make_tmap_4d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMbDqk, d->seq_k, d->batch, 1,
                      kv_st, 64, 128, true))
      return AF_ERR_INPUT;
    static bool attr = false;
    if (!attr) {
      if (set_smem(mla_bwd_scores_kernel, MlaScoresSmem::kTotal) != AF_OK) return AF_ERR_CUDA;
      attr = true;
    }
    ::af::note_launch();
    mla_bwd_scores_kernel<<<static_cast<unsigned>(k_tiles * bhs), 320, MlaScoresSmem::kTotal, s>>>(
        tq, tdo, tk, p);
    AF_CUDA_CHECK(cudaGetLastError());
  }

  {  // 2. dQ = dS' K  (N = 512, then the 64 rope columns)
    CUtensorMap tds, tkb;
    if (!tmap_3d(&tds, dsbuf, l.k_pad, l.q_pad, bhs, 64, 128) ||
        !make_tmap_4d(&tkb, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMbDqk, d->seq_k, d->batch, 1,
                      kv_st, 64, 64, true))
      return AF_ERR_INPUT;
    static bool attr = false;
    if (!attr) {
      if (set_smem(mla_bwd_gemm_kernel<false, 512>, MlaGemmSmem<512>::kTotal) != AF_OK ||
          set_smem(mla_bwd_gemm_kernel<false, 64>, MlaGemmSmem<64>::kTotal) != AF_OK)
        return AF_ERR_CUDA;
      attr = true;
    }
    const unsigned grid = static_cast<unsigned>(q_tiles * bhs);
    ::af::note_launch();
    mla_bwd_gemm_kernel<false, 512><<<grid, 192, MlaGemmSmem<512>::kTotal, s>>>(tds, tds, tkb, tkb,
                                                                               p, 0);
    AF_CUDA_CHECK(cudaGetLastError());
    ::af::note_launch();
    mla_bwd_gemm_kernel<false, 64><<<grid, 192, MlaGemmSmem<64>::kTotal, s>>>(tds, tds, tkb, tkb,
                                                                             p, 512);
    AF_CUDA_CHECK(cudaGetLastError());
  }

  {  // 3. dKV partials = sum_{h in group} dS'^T Q + P^T dO, then the group reduce
    CUtensorMap tds, tp, tqb, tdob;
    if (!tmap_3d(&tds, dsbuf, l.k_pad, l.q_pad, bhs, 64, 64) ||
        !tmap_3d(&tp, pbuf, l.k_pad, l.q_pad, bhs, 64, 64) ||
        !make_tmap_4d(&tqb, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMbDqk, d->seq_q, d->heads_q,
                      d->batch, d->q_stride, 64, 64, true) ||
        !make_tmap_4d(&tdob, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kMbDv, d->seq_q,
                      d->heads_q, d->batch, d->o_stride, 64, 64, true))
      return AF_ERR_INPUT;
    static bool attr = false;
    if (!attr) {
      if (set_smem(mla_bwd_gemm_kernel<true, 512>, MlaGemmSmem<512>::kTotal) != AF_OK ||
          set_smem(mla_bwd_gemm_kernel<true, 64>, MlaGemmSmem<64>::kTotal) != AF_OK)
        return AF_ERR_CUDA;
      attr = true;
    }
    const unsigned grid = static_cast<unsigned>(k_tiles * d->batch * l.groups);
    ::af::note_launch();
    mla_bwd_gemm_kernel<true, 512><<<grid, 192, MlaGemmSmem<512>::kTotal, s>>>(tds, tp, tqb, tdob,
                                                                              p, 0);
    AF_CUDA_CHECK(cudaGetLastError());
    ::af::note_launch();
    mla_bwd_gemm_kernel<true, 64><<<grid, 192, MlaGemmSmem<64>::kTotal, s>>>(tds, tp, tqb, tdob, p,
                                                                            512);
    AF_CUDA_CHECK(cudaGetLastError());
    const int64_t total = static_cast<int64_t>(d->batch) * d->seq_k * (kMbDqk / 4);
    ::af::note_launch();
    mla_bwd_reduce_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
        part, static_cast<int>(l.groups), d->batch, d->seq_k, static_cast<int>(l.k_pad),
        static_cast<__nv_bfloat16*>(dkv), d->k_stride[0], d->k_stride[2]);
    AF_CUDA_CHECK(cudaGetLastError());
  }
  return AF_OK;
}

}  // namespace af
