"""Kernel-dialect emission for the chosen B200 plan (inspection only).

The reference renders its assembled template as deterministic text (`lowering.code_generation`,
lowering.py:763-809: `kernel "<name>" template <kind> tile MxN { dims ...; buffer ...; grid ...
{ section ... } }`).  ``code_generation(spec)`` renders the same shape of text for what this
package actually launches for the spec on sm_100a: the hook family the planner chose, the
kernels, CTA shapes, shared-memory rings, TMEM column maps and the backward phases — so
``attnforge emit`` can report the real tile / stage / tier choices.  Pure host code, no GPU.
"""

from __future__ import annotations

from .plan import (ACT_IDENTITY, ACT_RELU, ACT_RELU2, ACT_SIGMOID, FAMILY_ABSSUM,
                   FAMILY_ELEMENTWISE, FAMILY_SOFTMAX, FM_NONE, plan_linear, plan_parallel)
from .spec import AttentionSpec, Pattern

_FAMILY = {FAMILY_SOFTMAX: "softmax", FAMILY_ELEMENTWISE: "elementwise", FAMILY_ABSSUM: "abssum"}
_ACT = {ACT_IDENTITY: "identity", ACT_SIGMOID: "sigmoid", ACT_RELU: "relu", ACT_RELU2: "relu2"}
_FM = {0: "none", 1: "silu", 2: "sigmoid", 3: "relu", 4: "tanh", 5: "exp"}


def _ceil(a: int, b: int) -> int:
    return (a + b - 1) // b


def _parallel(spec: AttentionSpec) -> list[str]:
    p = plan_parallel(spec)
    d = spec.dims
    dq, dv = d.d_qk, d.d_v
    bh = d.batch * d.heads
    lines = [f'kernel "{spec.name}" template parallel_online tile 128x128 target sm_100a {{',
             f"  dims batch={d.batch} heads={d.heads} heads_kv={d.kv_heads} seq_q={d.seq_q} "
             f"seq_k={d.seq_k} d_qk={dq} d_v={dv};"]
    band = p.band
    mask = ("none" if band.upper is None and band.window is None else
            f"band(upper={band.upper}, window={band.window})")
    hooks = (f"  lowering family={_FAMILY[p.family]} act={_ACT[p.act]} scale={p.scale:.6g} "
             f"mask={mask}")
    if p.cap_b:
        hooks += f" softcap={p.cap_a:g}*tanh({p.cap_b:g}*s)"
    if p.family == FAMILY_ELEMENTWISE and (p.slope_extra or p.slope_const):
        hooks += f" relpos_slope={p.slope_extra or p.slope_const} bias={p.bias:.6g}"
    if p.family == FAMILY_ABSSUM:
        hooks += (f" decay_mask={p.decay_extra}(gamma^(i-j), in-kernel) "
                  f"rownorm={'clamp(sum|s|,1,inf)' if p.normalize else 'none'}")
    maps = [f"{n}={_FM[m]}" for n, m in zip("qkv", (p.q_map, p.k_map, p.v_map)) if m != FM_NONE]
    if maps:
        hooks += " feature_maps=" + ",".join(maps)
    lines.append(hooks + ";")
    if spec.kv_shared and (dq, dv) == (576, 512):
        if d.seq_q == 1:
            lines += ["  kernel K3 mla_fwd_kernel<decode> cta 192 (4 softmax warps, TMA, MMA) "
                      "grid batch x splits x value_half;",
                      "  buffer q bf16[heads x 576]: cols [0,384) tmem (TS MMA A), [384,576) smem;",
                      "  buffer kv bf16[32 keys x 576] ring stages=4 (tma box 64x32, swizzle128);",
                      "  tmem S[0,64) double | Q[64,128) | O_half[128,384) | Q[384,512);",
                      "  combine mla_combine_kernel (LSE-weighted split merge);"]
        else:
            lines += ["  kernel K3 mla_fwd_kernel<prefill> cta 192 grid q_tiles x heads x "
                      "value_half;",
                      "  buffer q bf16[128 x 576]: cols [0,384) tmem (TS MMA A), [384,576) smem;",
                      "  buffer kv bf16[32 keys x 576] ring stages=4;",
                      "  tmem S[0,64) double | Q[64,128) | O_half[128,384) | Q[384,512);"]
    else:
        dv_k = min(dv, 128)
        stages = 1 if dq > 128 else 2
        warps = 8 if p.family == FAMILY_SOFTMAX else 16
        lines += [f"  kernel K1 parallel_fwd_kernel<{dq},{dv_k}> cta {32 * (warps + 2)} "
                  f"({warps} row warps, TMA, MMA) grid {_ceil(d.seq_q, 256)}x{bh}"
                  + (f" x {dv // 128} value slices" if dv > 128 else "") + ";",
                  f"  buffer q bf16[2x128 x {dq}] tier=smem stages=1 (tma box 64x128, "
                  "swizzle128);",
                  f"  buffer k bf16[128 x {dq}] tier=smem stages={stages};",
                  f"  buffer v bf16[128 x {dv_k}] tier=smem stages={stages};",
                  f"  tmem S0[0,128) S1[128,256) O0[256,{256 + dv_k}) O1[{256 + dv_k},"
                  f"{256 + 2 * dv_k});",
                  "  grid query_blocks {",
                  "    section load_q { tma q -> smem; }",
                  "    loop key_blocks (band-skipped) {",
                  "      section scores { tcgen05.mma S_t = Q_t K^T (SS, M128 N128) -> tmem; }",
                  f"      section fwd {{ row epilogue ({_FAMILY[p.family]}) P -> tmem bf16; }}",
                  "      section pv { tcgen05.mma O_t += P V (TS) ; }",
                  "    }",
                  "    section epilogue { tmem O -> registers -> bf16 global; row statistic; }",
                  "  }"]
    # backward
    if spec.kv_shared or (dq, dv) in ((192, 128), (128, 256)):
        lines += ["  backward materialised {",
                  "    section scores { K tile resident, Q/dO streamed; P, dS' -> HBM bf16; }",
                  "    section dq { tcgen05 GEMM dS' K (K-major A) ; }",
                  "    section dkv { tcgen05 GEMM dS'^T Q + P^T dO (MN-major A), head-group "
                  "partials, ordered reduce; }",
                  "  }"]
    else:
        lines += ["  backward atomic_free {",
                  "    kernel K2a parallel_bwd_dkdv_kernel cta 576 (16 row warps) grid key_tiles x "
                  "b*heads_kv "
                  "{ tmem S^T | dP^T | dV | dK; }",
                  "    kernel K2b parallel_bwd_dq_kernel cta 576 (16 row warps) grid q_tiles x b*heads "
                  "{ tmem S | dP | dQ | Q^A | dO^A; 64-key column halves; }",
                  "  }"]
    lines.append("}")
    return lines


def _linear(spec: AttentionSpec) -> list[str]:
    p = plan_linear(spec)
    d = spec.dims
    dk = 128 if d.d_qk <= 128 else 256
    dv = 128 if d.d_v <= 128 else 256
    lines = [f'kernel "{spec.name}" template recurrent_chunked tile 128x128 target sm_100a {{',
             f"  dims batch={d.batch} heads={d.heads} seq={d.seq_q} d_qk={d.d_qk} d_v={d.d_v} "
             f"(kernel {dk}/{dv});",
             f"  lowering q_scale={p.q_scale:.6g} decay={p.decay_const:g}"
             + "".join(f"*{n}" for n in p.decay_factors)
             + (f" key_gate={p.k_gate}" if p.k_gate else "")
             + (" factorised_decay" if p.decay_hint else "")
             + (f" v_map={_FM[p.v_map]}" if p.v_map else "") + ";",
             f"  kernel K4 linear_chunk_kernel<{dk}> cta 448 (8 row, 4 output, TMA+scan, MMA) "
             f"grid {d.batch * d.heads}x{dv // 64};",
             f"  buffer q,k bf16[128 x {dk}] ring stages={2 if dk == 128 else 1}; "
             f"v bf16[128 x 64] ring stages={3 if dk == 128 else 2};",
             f"  tmem S[0,128) OI[128,256) double QH[256,384) double H[384,{384 + 64 * dk // 128});",
             "  grid none {",
             "    loop chunks {",
             "      section scale { producer warp: cumsum log2 a (cp.async prefetch); }",
             "      section intra { S = Q K^T; P = S o D; O I = P V; }",
             "      section state { QH = Q H_in; H = g H + (K o w)^T V; }",
             "      section out { O = s (O I + cp Q H)  (output warps, one chunk behind); }",
             "    }",
             "  }",
             "  backward { three chunked runs (dQ fwd, dK rev, dV rev) + d log a scan; }",
             "  decode { af_linear_step: state <- a state + k^T v, o = q state; }",
             "}"]
    return lines


def code_generation(spec) -> str:
    """Deterministic text of the B200 plan for ``spec`` (the reference's ``emit`` output shape)."""
    from .api import _spec
    spec = _spec(spec)
    lines = _parallel(spec) if spec.pattern is Pattern.PARALLEL else _linear(spec)
    return "\n".join(lines) + "\n"
