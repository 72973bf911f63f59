// Elementwise hook programs on the GPU: the hooks of a variant that are evaluated on a whole
// tensor rather than fused into a template kernel's register epilogue —
//   output_mod        (attention.py:205; engine.py:502-504 parallel, 548-550 / 613-615 recurrent)
//   q_mod/k_mod/v_mod  that are not a compile-time scalar or one of af_feature_map's forms, e.g.
//                      ones that read per-step / per-head extras or the position grids
// — and their derivatives.  The host (hookvm.py) compiles the hook expression (exprlang grammar,
// docs/expression-language.md) into a postfix program; one thread evaluates the program for one
// element of the [B, H, S, D] output in fp32, carrying a forward-mode dual number so the same pass
// can also produce seed * d(hook)/d(operand `wrt`).  Derivative rules are the reference adjoints
// (graph.py:481-569): max/min ties to the first operand, abs' = sign with sign(0) = +1, clamp' = 1
// on the closed interval, where/comparisons carry no derivative into the condition.
#include <cuda_bf16.h>

#include <algorithm>

#include "host_common.h"

namespace af {
namespace {

enum HookOp : int32_t {
  kOpOperand = 1,  // + operand index
  kOpConst = 2,    // + const index
  kOpIndex = 3,    // + axis (0 b, 1 h, 2 s, 3 d): the element's coordinate as a value
  kOpNeg = 10, kOpAdd, kOpSub, kOpMul, kOpDiv,
  kOpExp = 20, kOpExp2, kOpLog, kOpAbs, kOpTanh, kOpSigmoid, kOpRelu, kOpSqrt,
  kOpMax = 30, kOpMin, kOpClamp, kOpWhere,
  kOpLt = 40, kOpLe, kOpGt, kOpGe, kOpEq, kOpNe,
};

constexpr int kStack = 16;

struct Dual {
  float v, d;
};

__device__ __forceinline__ float load_elem(const af_hook_operand& o, int64_t off) {
  if (o.dtype == AF_DTYPE_BF16)
    return __bfloat162float(static_cast<const __nv_bfloat16*>(o.ptr)[off]);
  return static_cast<const float*>(o.ptr)[off];
}

__device__ __forceinline__ void store_elem(const af_hook_operand& o, int64_t off, float v) {
  if (o.dtype == AF_DTYPE_BF16)
    static_cast<__nv_bfloat16*>(const_cast<void*>(o.ptr))[off] = __float2bfloat16_rn(v);
  else
    static_cast<float*>(const_cast<void*>(o.ptr))[off] = v;
}

__device__ __forceinline__ int64_t offset(const af_hook_operand& o, const int (&c)[4]) {
  return c[0] * o.stride[0] + c[1] * o.stride[1] + c[2] * o.stride[2] + c[3] * o.stride[3];
}

struct HookArgs {
  af_hook_program prog;
  af_hook_operand operand[AF_HOOK_MAX_OPERANDS];
  af_hook_operand seed, out, dout;
  int n_operands, wrt;
  int shape[4];
};

__global__ void __launch_bounds__(256) hook_eval_kernel(const __grid_constant__ HookArgs a) {
  const int64_t total =
      static_cast<int64_t>(a.shape[0]) * a.shape[1] * a.shape[2] * a.shape[3];
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int c[4];
    int64_t r = i;
    c[3] = static_cast<int>(r % a.shape[3]);
    r /= a.shape[3];
    c[2] = static_cast<int>(r % a.shape[2]);
    r /= a.shape[2];
    c[1] = static_cast<int>(r % a.shape[1]);
    c[0] = static_cast<int>(r / a.shape[1]);
    const float seed = a.wrt < 0 ? 0.0f : (a.seed.ptr != nullptr ? load_elem(a.seed, offset(a.seed, c))
                                                                 : 1.0f);
    Dual st[kStack];
    int sp = 0;
    for (int pc = 0; pc < a.prog.n_ops; ++pc) {
      const int op = a.prog.ops[pc];
      if (op == kOpOperand) {
        const int k = a.prog.ops[++pc];
        st[sp++] = {load_elem(a.operand[k], offset(a.operand[k], c)), k == a.wrt ? seed : 0.0f};
        continue;
      }
      if (op == kOpConst) {
        st[sp++] = {a.prog.consts[a.prog.ops[++pc]], 0.0f};
        continue;
      }
      if (op == kOpIndex) {
        st[sp++] = {static_cast<float>(c[a.prog.ops[++pc]]), 0.0f};
        continue;
      }
      if (op < kOpExp) {  // arithmetic
        if (op == kOpNeg) {
          st[sp - 1] = {-st[sp - 1].v, -st[sp - 1].d};
          continue;
        }
        const Dual y = st[--sp], x = st[sp - 1];
        Dual z;
        switch (op) {
          case kOpAdd: z = {x.v + y.v, x.d + y.d}; break;
          case kOpSub: z = {x.v - y.v, x.d - y.d}; break;
          case kOpMul: z = {x.v * y.v, x.d * y.v + x.v * y.d}; break;
          default: {  // kOpDiv: d(x/y) = dx/y - (x/y) dy / y
            const float q = x.v / y.v;
            z = {q, x.d / y.v - q * y.d / y.v};
          }
        }
        st[sp - 1] = z;
        continue;
      }
      if (op < kOpMax) {  // unary functions
        const Dual x = st[sp - 1];
        Dual z;
        switch (op) {
          case kOpExp: { const float e = expf(x.v); z = {e, x.d * e}; break; }
          case kOpExp2: { const float e = exp2f(x.v); z = {e, x.d * e * 0.6931471805599453f}; break; }
          case kOpLog: z = {logf(x.v), x.d / x.v}; break;
          case kOpAbs: z = {fabsf(x.v), x.v >= 0.0f ? x.d : -x.d}; break;
          case kOpTanh: { const float t = tanhf(x.v); z = {t, x.d * (1.0f - t * t)}; break; }
          case kOpSigmoid: { const float s = 1.0f / (1.0f + expf(-x.v)); z = {s, x.d * s * (1.0f - s)}; break; }
          case kOpRelu: z = {fmaxf(x.v, 0.0f), x.v >= 0.0f ? x.d : 0.0f}; break;
          default: { const float s = sqrtf(x.v); z = {s, x.d * 0.5f / s}; }  // kOpSqrt
        }
        st[sp - 1] = z;
        continue;
      }
      if (op == kOpClamp) {
        const Dual hi = st[--sp], lo = st[--sp], x = st[sp - 1];
        const bool inside = x.v >= lo.v && x.v <= hi.v;
        st[sp - 1] = {fminf(fmaxf(x.v, lo.v), hi.v), inside ? x.d : 0.0f};
        continue;
      }
      if (op == kOpWhere) {
        const Dual b = st[--sp], t = st[--sp], cnd = st[sp - 1];
        st[sp - 1] = cnd.v != 0.0f ? t : b;
        continue;
      }
      const Dual y = st[--sp], x = st[sp - 1];
      Dual z{0.0f, 0.0f};
      switch (op) {
        case kOpMax: z = x.v >= y.v ? x : y; break;
        case kOpMin: z = x.v <= y.v ? x : y; break;
        case kOpLt: z.v = x.v < y.v; break;
        case kOpLe: z.v = x.v <= y.v; break;
        case kOpGt: z.v = x.v > y.v; break;
        case kOpGe: z.v = x.v >= y.v; break;
        case kOpEq: z.v = x.v == y.v; break;
        default: z.v = x.v != y.v;  // kOpNe
      }
      st[sp - 1] = z;
    }
    if (a.out.ptr != nullptr) store_elem(a.out, offset(a.out, c), st[0].v);
    if (a.dout.ptr != nullptr) store_elem(a.dout, offset(a.dout, c), st[0].d);
  }
}

// Static check of the program: every opcode known, operands / constants / axes in range, the
// stack never underflows or exceeds kStack, and exactly one value remains.
bool program_ok(const af_hook_program* p, int n_operands) {
  if (p->n_ops < 1 || p->n_ops > AF_HOOK_MAX_OPS || p->n_consts < 0 ||
      p->n_consts > AF_HOOK_MAX_CONSTS)
    return false;
  int sp = 0;
  for (int pc = 0; pc < p->n_ops; ++pc) {
    const int op = p->ops[pc];
    int pop = 0, push = 1;
    if (op == kOpOperand || op == kOpConst || op == kOpIndex) {
      if (++pc >= p->n_ops) return false;
      const int x = p->ops[pc];
      if ((op == kOpOperand && (x < 0 || x >= n_operands)) ||
          (op == kOpConst && (x < 0 || x >= p->n_consts)) || (op == kOpIndex && (x < 0 || x > 3)))
        return false;
    } else if (op == kOpNeg || (op >= kOpExp && op <= kOpSqrt)) {
      pop = 1;
    } else if ((op >= kOpAdd && op <= kOpDiv) || op == kOpMax || op == kOpMin ||
               (op >= kOpLt && op <= kOpNe)) {
      pop = 2;
    } else if (op == kOpClamp || op == kOpWhere) {
      pop = 3;
    } else {
      return false;
    }
    if (sp < pop) return false;
    sp += push - pop;
    if (sp > kStack) return false;
  }
  return sp == 1;
}

}  // namespace
}  // namespace af

extern "C" int af_hook_eval(const af_hook_program* prog, const int32_t* shape,
                            const af_hook_operand* operands, int32_t n_operands, int32_t wrt,
                            const af_hook_operand* seed, const af_hook_operand* out,
                            const af_hook_operand* dout, void* stream) {
  using namespace af;
  AF_REQUIRE(prog != nullptr && shape != nullptr, AF_ERR_INPUT, "null program or shape");
  AF_REQUIRE(n_operands >= 0 && n_operands <= AF_HOOK_MAX_OPERANDS, AF_ERR_INPUT,
             "hook program takes at most %d operands (got %d)", AF_HOOK_MAX_OPERANDS, n_operands);
  AF_REQUIRE(program_ok(prog, n_operands), AF_ERR_INPUT, "malformed hook program");
  AF_REQUIRE(wrt >= -1 && wrt < n_operands, AF_ERR_INPUT, "derivative operand %d out of range",
             wrt);
  AF_REQUIRE(out != nullptr || dout != nullptr, AF_ERR_INPUT, "no output requested");
  AF_REQUIRE(dout == nullptr || wrt >= 0, AF_ERR_INPUT, "a derivative output needs wrt >= 0");
  HookArgs a{};
  a.prog = *prog;
  for (int k = 0; k < n_operands; ++k) {
    a.operand[k] = operands[k];
    AF_REQUIRE(operands[k].ptr != nullptr, AF_ERR_INPUT, "operand %d is null", k);
    AF_REQUIRE(operands[k].dtype == AF_DTYPE_BF16 || operands[k].dtype == AF_DTYPE_F32,
               AF_ERR_INPUT, "operand %d: unknown dtype", k);
  }
  a.n_operands = n_operands;
  a.wrt = wrt;
  if (seed != nullptr) a.seed = *seed;
  if (out != nullptr) a.out = *out;
  if (dout != nullptr) a.dout = *dout;
  int64_t total = 1;
  for (int i = 0; i < 4; ++i) {
    AF_REQUIRE(shape[i] >= 1, AF_ERR_SHAPE, "hook shape must be >= 1 on every axis");
    a.shape[i] = shape[i];
    total *= shape[i];
  }
  const int threads = 256;
  const unsigned blocks = static_cast<unsigned>(
      std::min<int64_t>((total + threads - 1) / threads, 32LL * sm_count()));
  ::af::note_launch();
  hook_eval_kernel<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}
