// Plain-old-data launch parameters shared by the host C-ABI and the kernels.
#pragma once
#include <cstdint>

namespace af {

// How a parallel-template variant's hooks were classified by the host lowering
// (paper_2502_15349_b200/plan.py).  Each family is one register-level epilogue.
enum Family : int {
  kFamilySoftmax = 0,      // online softmax rownorm (attention.py:556-572)
  kFamilyElementwise = 1,  // score mods only, no rownorm (sigmoid / relu / identity)
  kFamilyAbssum = 2,       // retention-parallel: causal decay mask gamma_h^(i-j) (slope[h] holds
                           // log2 gamma_h) and rows / clamp(sum |s|, 1, inf) when cap_a != 0
                           // (attention.py:575-586, 600-671)
};

enum Act : int {
  kActIdentity = 0,
  kActSigmoid = 1,
  kActRelu = 2,
  kActRelu2 = 3,  // relu(z)^2 (squared-relu variant; post-scales folded into z by the planner)
  kActSoftcap = 4,  // softmax family: z -> cap_a tanh(cap_b z) ahead of the softmax
};

// Band mask derived from the variant's mask_mod expressions:
//   keep (i, j)  iff  j < seq_k
//                and (!causal || j <= i + diag_offset)
//                and (window <= 0 || i + diag_offset - j < window)
struct MaskParams {
  int causal;
  int diag_offset;
  int window;
};

struct ParallelFwdParams {
  int batch, heads_q, heads_kv, seq_q, seq_k, d_qk, d_v;
  float scale;       // q_mod scale folded into the scores (e.g. 1/sqrt(d_qk))
  float scale_log2;  // scale * log2(e)
  MaskParams mask;
  // elementwise family: z = scale*qk - slope[h]*(i - j) + bias ; p = act(z)
  int act;
  const float* slope;  // per q-head slope (may be null)
  float bias;
  float cap_a, cap_b;  // softmax soft-cap (kActSoftcap): z -> cap_a tanh(cap_b z)
  // output O (bf16) with element strides, LSE fp32 [B, Hq, Sq] (may be null)
  void* o;
  int64_t o_stride_b, o_stride_h, o_stride_s;
  float* lse;
  int o_tma;  // 1: O leaves through the kernel's O tensor map (TMA stores of staged boxes)
};

struct ParallelBwdParams {
  int batch, heads_q, heads_kv, seq_q, seq_k, d_qk, d_v;
  float scale, scale_log2;
  MaskParams mask;
  int act;
  const float* slope;
  float bias;
  float cap_a, cap_b;  // softmax soft-cap (kActSoftcap)
  const float* lse;    // [B, Hq, Sq] natural-log LSE (softmax family)
  const float* delta;  // [B, Hq, Sq] rowsum(dO*O) (softmax family)
  float* dq_accum;     // [B, Hq, Sq, Dqk] fp32 accumulator (zeroed)
  void* dk;            // [B, Hkv, Sk, Dqk] bf16 (group-summed)
  void* dv;            // [B, Hkv, Sk, Dv] bf16 (group-summed)
  int64_t dk_stride_b, dk_stride_h, dk_stride_s;
  int64_t dv_stride_b, dv_stride_h, dv_stride_s;
  int dkv_tma;  // fused kernel: dK / dV leave through its tensor maps (TMA stores)
};

}  // namespace af
