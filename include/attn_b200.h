/*
 * attn_b200 — C ABI of the B200 (sm_100a) attention-template kernels.
 *
 * This is the drop-in boundary for the hot path of the attnforge reference (AttentionEngine,
 * arXiv 2502.15349).  Each entry point replaces one reference executor; the host lowering
 * (paper_2502_15349_b200/plan.py) turns an AttentionSpec into the descriptor structs below.
 * Plain pointers and sizes only: device pointers are CUDA global-memory addresses, `stream` is a
 * cudaStream_t (NULL = legacy default stream).  All calls are stream-ordered and asynchronous;
 * outputs are caller-allocated.  Nothing here owns memory between calls.
 *
 * Status codes mirror attnforge/errors.py kinds (errors.py:30-82): AF_ERR_INPUT* map to
 * InputError subclasses (CLI exit 2), AF_ERR_UNSUPPORTED / AF_ERR_NAN to SemanticError (exit 1).
 */
#ifndef ATTN_B200_H_
#define ATTN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py kinds) ---- */
enum {
  AF_OK = 0,
  AF_ERR_INPUT = 1,          /* InputError            kind "input"          */
  AF_ERR_SHAPE = 2,          /* ShapeError            kind "shape-mismatch" */
  AF_ERR_UNSUPPORTED = 3,    /* UnsupportedError      kind "unsupported"    */
  AF_ERR_NAN = 4,            /* NanError              kind "nan-in-output"  */
  AF_ERR_CUDA = 5,           /* launch / driver failure (no reference analogue) */
};

/* ---- parallel template (attention.py:389-449, engine.py:423-505) ---- */
enum { AF_FAMILY_SOFTMAX = 0, AF_FAMILY_ELEMENTWISE = 1, AF_FAMILY_ABSSUM = 2 };
enum { AF_ACT_IDENTITY = 0, AF_ACT_SIGMOID = 1, AF_ACT_RELU = 2, AF_ACT_RELU2 = 3 };
enum { AF_DTYPE_BF16 = 0, AF_DTYPE_F32 = 1 };

typedef struct af_parallel_desc {
  int32_t batch, heads_q, heads_kv, seq_q, seq_k, d_qk, d_v;
  int32_t dtype;             /* AF_DTYPE_BF16 (tcgen05 path) or AF_DTYPE_F32 (exact FFMA path) */
  /* element strides [b, h, s, d] of q, k, v, o (d stride must be 1) */
  int64_t q_stride[4], k_stride[4], v_stride[4], o_stride[4];
  int32_t family;            /* AF_FAMILY_*: classified online_func / score_mod hook family */
  int32_t act;               /* AF_ACT_*: elementwise score activation (elementwise family) */
  float scale;               /* q_mod scale folded into scores, e.g. 1/sqrt(d_qk)          */
  int32_t causal;            /* band mask from mask_mod: keep j <= i + diag_offset         */
  int32_t diag_offset;
  int32_t window;            /* >0: also keep only i + diag_offset - j < window            */
  const float* slope;        /* elementwise family: z -= slope[h] * (i - j); may be NULL.
                                abssum family: log2 gamma_h of the causal decay mask
                                z = tau q.k gamma_h^(i-j) [j <= i]                          */
  float bias;                /* elementwise family: z += bias                               */
  float cap_a, cap_b;        /* softmax family soft-cap z -> cap_a * tanh(cap_b * z); cap_b = 0
                                disables it (capped-softmax variant: 30 * tanh(z / 30)).
                                abssum family: cap_a = 1 divides rows by clamp(sum|z|, 1, inf)
                                (retention-parallel), 0 leaves them unnormalised; lse then
                                receives the row abs-sum                                     */
  /* tile configuration (0 = the library's default; schedule.py's measured mode picks others,
   * replacing the reference's analytic tile scheduler, scheduling.py:256-266) */
  int32_t kv_stages;         /* K1 K/V ring depth for head dims <= 128: 1 or 2 (default 2)   */
  int32_t head_groups;       /* materialised backward: query-head chunks of the key-side GEMMs
                                (default: enough CTAs for ~4 waves)                          */
  int32_t bwd_mode;          /* backward kernels for head dims 128/128: AF_BWD_DEFAULT (fused),
                                AF_BWD_SPLIT (K2a + K2b: S and dP recomputed, bitwise
                                deterministic), AF_BWD_FUSED (one 5-GEMM kernel, dQ reduced
                                through L2 in fp32: deterministic to fp32 rounding only)      */
} af_parallel_desc;
enum { AF_BWD_DEFAULT = 0, AF_BWD_SPLIT = 1, AF_BWD_FUSED = 2 };

/* O = template_forward(q, k, v); lse[b,h,i] = log-sum-exp of row i (softmax family, may be NULL).
 * Replaces engine.run_tiled_parallel (engine.py:423) / lowering.ExecutablePlan.run (lowering.py:857). */
int af_parallel_fwd(const af_parallel_desc* desc, const void* q, const void* k, const void* v,
                    void* o, float* lse, void* stream);

/* Bytes of device scratch af_parallel_bwd needs (row statistics; + the fp32 dQ accumulator on the
 * fused path). */
size_t af_parallel_bwd_workspace(const af_parallel_desc* desc);

/* VJP of af_parallel_fwd for cotangent dO (bf16).  dq/dk/dv use the q/k/v strides of desc; dk/dv
 * are summed over the query heads of each GQA group.  MLA lowering ((d_qk, d_v) = (576, 512),
 * heads_kv = 1, v == k): dk receives the latent-cache gradient dK + [dV, 0] and dv is unused.  Replaces engine.autodiff_grads
 * (engine.py:630) over attention.build_parallel (attention.py:389) with seed dO. */
int af_parallel_bwd(const af_parallel_desc* desc, const void* q, const void* k, const void* v,
                    const void* o, const float* lse, const void* dout, void* dq, void* dk,
                    void* dv, void* workspace, size_t workspace_bytes, void* stream);

/* ---- linear / recurrent template (attention.py:455-511, engine.py:525-616) ---- */
/* Per-step tensors are fp32 with element strides [b, h, s] (0 = broadcast).  The h_mod of the
 * variant factors as h * a_t (attention.diagonal_scale, attention.py:332-369) with
 *   a_t = exp(log_decay_const) * prod_f decay_factor[f][b, h, t]          (n_decay_factors <= 2)
 * and k_mod = k * key_gate[b, h, t] (key_gate may be NULL). */
typedef struct af_linear_desc {
  int32_t batch, heads, seq, d_k, d_v;
  int32_t chunk;             /* chunk length of the intra/inter decomposition (128) */
  float q_scale;             /* q_mod scale (e.g. 1/sqrt(d_k)); 1 when absent       */
  /* element strides [b, h, s, d] of q, k, v, o (o also describes dout / dq layouts) */
  int64_t q_stride[4], k_stride[4], v_stride[4], o_stride[4];
  float log_decay_const;
  int32_t n_decay_factors;
  const float* decay_factor[2];
  int64_t decay_factor_stride[2][3];
  const float* key_gate;
  int64_t key_gate_stride[3];
  int32_t decay_hint;        /* 1: the per-step decay is expected to stay mild (constant fills such
                                as RetNet's gamma_h >= 0.5), enabling the factorised-decay kernel
                                variant (still checked per chunk at run time); 0: generic */
} af_linear_desc;

/* Bytes of device scratch af_linear_fwd needs (the per-chunk decay scan shared by the passes). */
size_t af_linear_fwd_workspace(const af_linear_desc* desc);

/* o_t = q_scale * q_t h_t,  h_t = a_t h_{t-1} + (k_t * gate_t)^T v_t,  h_0 = 0.
 * final_state (may be NULL): fp32 [B, H, d_k, d_v] receives h_S, the state after the last token.
 * Replaces engine.run_chunk_recurrent (engine.py:554). */
int af_linear_fwd(const af_linear_desc* desc, const void* q, const void* k, const void* v,
                  void* o, float* final_state, void* workspace, size_t workspace_bytes,
                  void* stream);

/* One generation step (desc->seq == 1): state <- a_t state + (k_t * gate_t)^T v_t (fp32
 * [B, H, d_k, d_v], in place), o_t = q_scale * q_t state.  The body of engine.run_step_recurrent
 * (engine.py:539-547) for a carried state, e.g. af_linear_fwd's final_state of the prompt. */
int af_linear_step(const af_linear_desc* desc, const void* q, const void* k, const void* v,
                   float* state, void* o, void* stream);

size_t af_linear_bwd_workspace(const af_linear_desc* desc);

/* VJP of af_linear_fwd for cotangent dout: dq, dk (w.r.t. the raw k), dv (bf16, q/k/v strides)
 * and, when non-NULL, d_decay_factor[f] / d_key_gate (fp32, ACCUMULATED with the strides of the
 * corresponding input — zero them first; broadcast axes sum).  Replaces engine.autodiff_grads
 * over RecurrenceDef.unroll (attention.py:468). */
int af_linear_bwd(const af_linear_desc* desc, const void* q, const void* k, const void* v,
                  const void* dout, void* dq, void* dk, void* dv, float* const* d_decay_factor,
                  float* d_key_gate, void* workspace, size_t workspace_bytes, void* stream);

/* ---- MLA decode (softmax over a shared latent cache; V = first d_v columns of K) ---- */
typedef struct af_mla_desc {
  int32_t batch, heads, seq_k, d_qk, d_v;
  float scale;
  int32_t splits;            /* KV splits per (batch, value half); 0 = minimise waves x blocks */
} af_mla_desc;

size_t af_mla_decode_workspace(const af_mla_desc* desc);

/* q [B, H, d_qk] bf16, kv [B, seq_k, d_qk] bf16 -> o [B, H, d_v] bf16, lse [B, H] fp32.
 * Replaces engine.run_tiled_parallel with seq_q = 1 (test_engine.py:224-230). */
int af_mla_decode(const af_mla_desc* desc, const void* q, const void* kv, void* o, float* lse,
                  void* workspace, size_t workspace_bytes, void* stream);

/* ---- feature maps (q_mod / k_mod / v_mod that are a function of the tensor alone) ---- */
enum { AF_FM_NONE = 0, AF_FM_SILU = 1, AF_FM_SIGMOID = 2, AF_FM_RELU = 3, AF_FM_TANH = 4,
       AF_FM_EXP = 5 };

/* y = f(x) (backward = 0) or y = dy * f'(x) (backward = 1) over n contiguous bf16 elements
 * (n a multiple of 8).  Applied ahead of the template kernels; replaces the per-tile evaluation
 * of the mod hooks in engine._premod_qkv (engine.py:511-522) / build_parallel. */
int af_feature_map(int kind, int backward, const void* x, const void* dy, void* y, int64_t n,
                   void* stream);

/* ---- elementwise hook programs (output_mod, general q/k/v mods) ---- */
/* A hook expression compiled by the host (paper_2502_15349_b200/hookvm.py) into a postfix program
 * evaluated per element of a [B, H, S, D] tensor in fp32 with a forward-mode dual number.
 * Opcodes: 1 operand <k>, 2 const <i>, 3 index <axis>; 10 neg, 11 add, 12 sub, 13 mul, 14 div;
 * 20 exp, 21 exp2, 22 log, 23 abs, 24 tanh, 25 sigmoid, 26 relu, 27 sqrt; 30 max, 31 min,
 * 32 clamp, 33 where; 40 lt, 41 le, 42 gt, 43 ge, 44 eq, 45 ne.  Derivatives follow the reference
 * adjoint rules (graph.py:481-569). */
#define AF_HOOK_MAX_OPS 128
#define AF_HOOK_MAX_CONSTS 32
#define AF_HOOK_MAX_OPERANDS 8
typedef struct af_hook_program {
  int32_t n_ops;
  int32_t ops[AF_HOOK_MAX_OPS];
  int32_t n_consts;
  float consts[AF_HOOK_MAX_CONSTS];
} af_hook_program;

/* A bf16 / fp32 tensor seen as [B, H, S, D] with element strides (0 = broadcast axis). */
typedef struct af_hook_operand {
  const void* ptr;
  int32_t dtype;             /* AF_DTYPE_BF16 or AF_DTYPE_F32 */
  int64_t stride[4];
} af_hook_operand;

/* out[i] = hook(operands)[i]  and/or  dout[i] = seed[i] * d hook / d operand[wrt] at i (seed NULL
 * = 1) over the element grid `shape` [B, H, S, D].  Replaces the per-tile evaluation of
 * output_mod (engine.py:502-504, 548-550) and of extra-reading q/k/v mods (engine.py:511-522); the
 * derivative output gives the VJP through the hook (graph.py:436-591). */
int af_hook_eval(const af_hook_program* prog, const int32_t* shape,
                 const af_hook_operand* operands, int32_t n_operands, int32_t wrt,
                 const af_hook_operand* seed, const af_hook_operand* out,
                 const af_hook_operand* dout, void* stream);

/* ---- materialised tier of the parallel template (engine.run_naive_parallel on the GPU) ---- */
/* For variants the fused kernels do not lower: S = Qm Km^T and O = P Vm are plain GEMMs, the
 * score hooks run through af_hook_eval over [B, H, Sq, Sk], and these apply the recognised row
 * normalisation to contiguous fp32 score rows [rows, n]. */
enum { AF_ROWNORM_NONE = 0, AF_ROWNORM_SOFTMAX = 1, AF_ROWNORM_ABSSUM = 2 };

/* p = rownorm(z); stat = LSE (softmax; -inf for fully-masked rows) or the row abs-sum (abssum).
 * attention.py:556-586. */
int af_rownorm_fwd(int32_t kind, const float* z, float* p, float* stat, int64_t rows, int64_t n,
                   void* stream);

/* dz = d rownorm / dz applied to dp, given rowdot = <dO, O> per row (graph.py:436-591 rules). */
int af_rownorm_bwd(int32_t kind, const float* z, const float* p, const float* dp,
                   const float* rowdot, const float* stat, float* dz, int64_t rows, int64_t n,
                   void* stream);

/* out[b, h, s] = sum_d a[b, h, s, d] * b[b, h, s, d] (the softmax VJP's row term). */
int af_rowdot(const af_hook_operand* a, const af_hook_operand* b, const int32_t* shape,
              float* out, void* stream);

/* ---- diagnostics ---- */
const char* af_status_string(int status);
const char* af_last_error(void);      /* thread-local message of the last failing call */
int af_device_sm_count(void);
uint64_t af_launch_count(void);   /* kernels this library has launched (process-wide) */

#ifdef __cplusplus
}
#endif
#endif /* ATTN_B200_H_ */
