"""GPU executors with the reference's call signatures (the drop-in boundary, Python side).

Every function takes an ``AttentionSpec`` (this package's, or an ``attnforge`` one — converted by
``spec.from_reference``) and a dict of CUDA tensors named like the reference's ``arrays``
(``q``, ``k``, ``v`` and each extra; ``qidx``/``kidx`` are synthesised in-kernel and ignored), and
returns freshly allocated CUDA tensors.  Inputs are never mutated.

========================================  =====================================================
reference (attnforge)                     here
========================================  =====================================================
engine.run_tiled_parallel  (engine.py:423)  ``run_tiled_parallel`` / ``parallel_forward`` (+LSE)
engine.run_naive_parallel  (engine.py:401)  ``run_naive_parallel`` (same kernel; tiled ≡ naive)
engine.run_chunk_recurrent (engine.py:554)  ``run_chunk_recurrent`` / ``linear_forward``
engine.run_step_recurrent  (engine.py:525)  ``run_step_recurrent`` (chunked kernel; chunk ≡ step)
engine.autodiff_grads      (engine.py:630)  ``autodiff_grads`` (seed ones, or an explicit ``dout``)
ExecutablePlan.run         (lowering.py:857) ``bind(spec).run(arrays)``
========================================  =====================================================

There is no CPU path: every call lowers the spec (``plan.py``) and launches the sm_100a library
through its C ABI (``runtime.py``); if the library or a GPU is missing the call raises.
"""

from __future__ import annotations

import contextlib
import contextvars
import dataclasses
import math
from dataclasses import dataclass

import torch

from . import generic
from . import hookvm
from . import runtime as rt
from .errors import InputError, NanError, ShapeError, UnsupportedError
from .plan import (FAMILY_ABSSUM, FAMILY_SOFTMAX, FM_HOOK, LinearPlan, ParallelPlan, plan_linear,
                   plan_parallel)
from .spec import AttentionSpec, Pattern, from_reference

_BF16 = torch.bfloat16


# Output-buffer reuse for repeated same-shape calls (HostPipeline slots): inside
# ``reuse_buffers(cache)`` the executors' output / workspace tensors come from ``cache`` (keyed by
# allocation site) instead of fresh allocations; the caller owns the ordering of reuse.
_REUSE: contextvars.ContextVar = contextvars.ContextVar("af_reuse_buffers", default=None)


@contextlib.contextmanager
def reuse_buffers(cache: dict):
    token = _REUSE.set(cache)
    try:
        yield cache
    finally:
        _REUSE.reset(token)


def _empty(key: str, shape, dtype, device) -> torch.Tensor:
    cache = _REUSE.get()
    shape = tuple(int(x) for x in shape)
    if cache is None:
        return torch.empty(shape, dtype=dtype, device=device)
    ck = (key, shape, dtype, str(device))  # several chunk widths may share one cache
    t = cache.get(ck)
    if t is None:
        t = torch.empty(shape, dtype=dtype, device=device)
        cache[ck] = t
    return t


_TUNE: contextvars.ContextVar = contextvars.ContextVar("af_tuning", default=None)


@contextlib.contextmanager
def tuned(config: dict):
    """Launch with an explicit tile configuration (schedule.Candidate fields) inside the block —
    what the measured scheduler's ``measure`` uses to time one candidate."""
    token = _TUNE.set(dict(config))
    try:
        yield
    finally:
        _TUNE.reset(token)


def _tuning(spec) -> dict:
    t = _TUNE.get()
    if t is not None:
        return t
    from . import schedule
    return schedule.tuning(spec)


def _spec(spec) -> AttentionSpec:
    return spec if isinstance(spec, AttentionSpec) else from_reference(spec)


def _stream() -> int | None:
    return torch.cuda.current_stream().cuda_stream


def _need(arrays: dict, name: str) -> torch.Tensor:
    if name not in arrays:
        raise InputError("missing input tensor", name=name)
    t = arrays[name]
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InputError("inputs must be CUDA tensors (this backend has no CPU path)", name=name)
    return t


def _check_shape(t: torch.Tensor, want: tuple, name: str) -> None:
    if tuple(t.shape) != tuple(want):
        raise ShapeError("input shape mismatch", name=name, want=tuple(want), got=tuple(t.shape))


def _as(t: torch.Tensor, dtype) -> torch.Tensor:
    t = t if t.dtype == dtype else t.to(dtype)
    return t if t.stride(-1) == 1 else t.contiguous()


def _check_nan(out: torch.Tensor, what: str) -> torch.Tensor:
    if torch.isnan(out).any().item():
        raise NanError("output contains NaN", path=what, count=int(torch.isnan(out).sum()))
    return out


# ───────────────────────────── feature maps ─────────────────────────────

def _fmap(kind: int, x: torch.Tensor, dy: torch.Tensor | None = None) -> torch.Tensor:
    """f(x) (or dy * f'(x)) for an elementwise q/k/v feature map, on the GPU
    (``af_feature_map``); bf16 in and out."""
    if kind == 0:
        return x if dy is None else dy
    shape = x.shape
    xf = _as(x, _BF16).contiguous().reshape(-1)
    n = xf.numel()
    pad = (-n) % 8
    if pad:
        xf = torch.nn.functional.pad(xf, (0, pad))
    gf = None
    if dy is not None:
        gf = _as(dy, _BF16).contiguous().reshape(-1)
        if pad:
            gf = torch.nn.functional.pad(gf, (0, pad))
    y = torch.empty_like(xf)
    rt.check(rt.lib().af_feature_map(int(kind), int(dy is not None), xf.data_ptr(),
                                     rt.ptr(gf), y.data_ptr(), xf.numel(), _stream()),
             "af_feature_map")
    return y[:n].reshape(shape)


def _maps(plan) -> tuple[int, int, int]:
    return getattr(plan, "q_map", 0), getattr(plan, "k_map", 0), getattr(plan, "v_map", 0)


def _hook_tensors(plan, arrays: dict, **named) -> dict:
    """Operands a compiled hook may read: the spec's extras (as given) plus ``named``."""
    out = {e.name: arrays[e.name] for e in plan.spec.extra_inputs if e.name in arrays}
    out.update(named)
    return out


def _mod(plan, var: str, x: torch.Tensor, arrays: dict) -> torch.Tensor:
    """q_mod / k_mod / v_mod applied ahead of the template kernels: af_feature_map for its fixed
    forms, a compiled hook program (af_hook_eval) for any other elementwise mod."""
    kind = getattr(plan, f"{var}_map", 0)
    if kind == FM_HOOK:
        return hookvm.run_hook(plan.hooks[var], x.shape, _hook_tensors(plan, arrays, **{var: x}),
                               out_dtype=_BF16)[0]
    return _fmap(kind, x)


def _hook_extra_grads(plan, key: str, shape, tensors: dict, seed: torch.Tensor,
                      grads_x: dict) -> None:
    """Accumulate seed * d hook / d extra (summed over the extra's broadcast axes) for every
    differentiable extra the hook reads."""
    hook = plan.hooks[key]
    for e in plan.spec.extra_inputs:
        if e.differentiable and hook.uses(e.name):
            _, de = hookvm.run_hook(hook, shape, tensors, value=False, wrt=e.name, seed=seed)
            de = hookvm.sum_to(de, tuple(tensors[e.name].shape))
            grads_x[e.name] = de if e.name not in grads_x else grads_x[e.name] + de


def _mod_vjp(plan, var: str, x: torch.Tensor, g: torch.Tensor, arrays: dict,
             grads_x: dict) -> torch.Tensor:
    """dL/dx from dL/d mod(x); extras read by a hook mod receive their gradient in grads_x."""
    kind = getattr(plan, f"{var}_map", 0)
    if kind == FM_HOOK:
        tensors = _hook_tensors(plan, arrays, **{var: x})
        _, dx = hookvm.run_hook(plan.hooks[var], x.shape, tensors, value=False, wrt=var, seed=g,
                                deriv_dtype=_BF16)
        _hook_extra_grads(plan, var, x.shape, tensors, g, grads_x)
        return dx
    return _fmap(kind, x, g)


def _out_mod(plan, o: torch.Tensor, arrays: dict) -> torch.Tensor:
    """output_mod on the full output (engine.py:502-504, 548-550, 613-615)."""
    if "o" not in plan.hooks:
        return o
    return hookvm.run_hook(plan.hooks["o"], o.shape, _hook_tensors(plan, arrays, o=o),
                           out_dtype=o.dtype)[0]


def _out_mod_vjp(plan, o_inner: torch.Tensor, dout: torch.Tensor, arrays: dict,
                 grads_x: dict) -> torch.Tensor:
    tensors = _hook_tensors(plan, arrays, o=o_inner)
    _, d = hookvm.run_hook(plan.hooks["o"], o_inner.shape, tensors, value=False, wrt="o",
                           seed=dout, deriv_dtype=_BF16)
    _hook_extra_grads(plan, "o", o_inner.shape, tensors, dout, grads_x)
    return d


def _check_extra_grads(spec, arrays) -> None:
    """Differentiable extras get gradients on the materialised tier and through whole-tensor hook
    programs; one read by a fused kernel's score epilogue (a relative-position slope, the
    declared decay mask) raises — its gradient is not lowered there."""
    route, plan = route_parallel(spec, arrays)
    if route == "generic":
        return
    hook_only = _hook_only_extras(plan)
    for e in spec.extra_inputs:
        if e.differentiable and e.name not in hook_only:
            raise UnsupportedError("gradients w.r.t. extras read by the fused score hooks are "
                                   "not lowered", extra=e.name)


def _hook_only_extras(plan) -> set:
    """Differentiable extras read only by whole-tensor hooks (their gradients are lowered)."""
    return {e.name for e in plan.spec.extra_inputs
            if e.differentiable and any(h.uses(e.name) for h in plan.hooks.values())}


# ───────────────────────────── parallel template ─────────────────────────────

def _parallel_inputs(plan: ParallelPlan, arrays: dict, dtype):
    d = plan.spec.dims
    hkv = d.kv_heads
    q = _need(arrays, "q")
    k = _need(arrays, "k")
    _check_shape(q, (d.batch, d.heads, d.seq_q, d.d_qk), "q")
    _check_shape(k, (d.batch, hkv, d.seq_k, d.d_qk), "k")
    if plan.spec.kv_shared:
        v = k[..., : d.d_v]
    else:
        v = _need(arrays, "v")
        _check_shape(v, (d.batch, hkv, d.seq_k, d.d_v), "v")
    slope = None
    if plan.family == FAMILY_ABSSUM:
        _check_decay_mask(plan, _need(arrays, plan.decay_extra), q.device)
        slope = torch.tensor([math.log2(g) for g in plan.decay_gammas], device=q.device,
                             dtype=torch.float32)
    elif plan.slope_extra is not None:
        slope = _need(arrays, plan.slope_extra).to(torch.float32).reshape(-1)
        slope = slope.expand(d.heads).contiguous() if slope.numel() == 1 else slope.contiguous()
    elif plan.slope_const != 0.0:
        slope = torch.full((d.heads,), plan.slope_const, device=q.device, dtype=torch.float32)
    qm, km, vm = _maps(plan)
    if qm or km or vm:
        if dtype != _BF16 or plan.spec.kv_shared:
            raise UnsupportedError("feature maps run on the bf16 path of non-MLA variants only")
        q, k, v = (_mod(plan, n, t, arrays) for n, t in (("q", q), ("k", k), ("v", v)))
    return _as(q, dtype), _as(k, dtype), _as(v, dtype), slope


def _desc(plan: ParallelPlan, q, k, v, o, slope, dtype_code: int) -> rt.ParallelDesc:
    d = plan.spec.dims
    c = rt.ParallelDesc()
    c.batch, c.heads_q, c.heads_kv = d.batch, d.heads, d.kv_heads
    c.seq_q, c.seq_k = d.seq_q, d.seq_k
    c.d_qk, c.d_v = int(q.shape[-1]), int(v.shape[-1])  # kernel (possibly padded) head dims
    c.dtype = dtype_code
    c.q_stride, c.k_stride, c.v_stride = rt.strides4(q), rt.strides4(k), rt.strides4(v)
    c.o_stride = rt.strides4(o)
    c.family, c.act, c.scale = plan.family, plan.act, float(plan.scale)
    c.causal, c.diag_offset, c.window = plan.band.causal, plan.band.diag_offset, \
        plan.band.kernel_window
    c.slope = rt.ptr(slope)
    c.bias = float(plan.bias)
    c.cap_a, c.cap_b = float(plan.cap_a), float(plan.cap_b)
    if plan.family == FAMILY_ABSSUM:  # cap_a = 1: rows divided by clamp(sum |s|, 1, inf)
        c.cap_a, c.cap_b = (1.0 if plan.normalize else 0.0), 0.0
    t = _tuning(plan.spec)
    c.kv_stages, c.head_groups = int(t.get("kv_stages", 0)), int(t.get("head_groups", 0))
    c.bwd_mode = rt.AF_BWD_SPLIT if _DETERMINISTIC[0] else int(t.get("bwd_mode", 0))
    return c


# Bitwise-deterministic backward (the reference's SPEC.md:335 contract): the fused 5-GEMM backward
# adds dQ partials of different key tiles in L2 arrival order (fp32), so it is reproducible to
# fp32 rounding only; deterministic mode selects the split K2a/K2b kernels (S and dP recomputed).
_DETERMINISTIC = [False]


def use_deterministic_backward(flag: bool = True) -> None:
    """Select the bitwise-deterministic backward kernels for every later call (default off)."""
    _DETERMINISTIC[0] = bool(flag)


def deterministic_backward() -> bool:
    return _DETERMINISTIC[0]


_MASK_CHECKED: dict = {}


def _check_decay_mask(plan: ParallelPlan, mask: torch.Tensor, device) -> None:
    """The abssum kernels synthesise the causal decay mask gamma_h^(i-j) in-register from the
    extra's declared fill; a mask tensor holding anything else is not lowered.  Checked once per
    tensor version (a GPU pass over the mask)."""
    d = plan.spec.dims
    key = (mask.data_ptr(), mask._version, tuple(mask.shape), plan.decay_gammas)
    if _MASK_CHECKED.get(key):
        return
    _check_shape(mask, (1, d.heads, d.seq_q, d.seq_k), plan.decay_extra)
    i = torch.arange(d.seq_q, device=device, dtype=torch.float64).view(1, 1, -1, 1)
    j = torch.arange(d.seq_k, device=device, dtype=torch.float64).view(1, 1, 1, -1)
    g = torch.tensor(plan.decay_gammas, device=device, dtype=torch.float64).view(1, -1, 1, 1)
    want = torch.where(i >= j, g ** (i - j).clamp(min=0), torch.zeros((), device=device,
                                                                        dtype=torch.float64))
    err = (mask.to(device=device, dtype=torch.float64) - want).abs().max().item()
    if not err <= 1e-6:
        raise UnsupportedError("decay-mask extra differs from its declared causal_decay_mask "
                               "fill; arbitrary materialised score masks are not lowered",
                               extra=plan.decay_extra, max_abs_diff=err)
    if len(_MASK_CHECKED) > 64:
        _MASK_CHECKED.clear()
    _MASK_CHECKED[key] = True


MLA_DQK, MLA_DV = 576, 512
_KERNEL_DIMS = ((64, 64), (128, 128), (192, 128))


def _padded_dim(spec, precision: str) -> int | None:
    """Head dims the bf16 tcgen05 kernels are not instantiated for (e.g. the reference's
    16/32-wide variant files) run zero-padded to 64 or 128: zero q/k columns add nothing to
    Q K^T, zero v columns only produce output columns that are sliced off, and the q_mod scale
    was already fixed from the spec's own dims.  None = run as is."""
    d = spec.dims
    if precision != "bf16" or spec.kv_shared or (d.d_qk, d.d_v) in _KERNEL_DIMS:
        return None
    m = max(d.d_qk, d.d_v)
    if m > 128:
        return None
    return 64 if m <= 64 else 128


def _pad_last(t: torch.Tensor, n: int) -> torch.Tensor:
    return t if t.shape[-1] == n else torch.nn.functional.pad(t, (0, n - t.shape[-1]))


def mla_decode(q: torch.Tensor, kv: torch.Tensor, scale: float, splits: int = 0):
    """K3 decode: softmax attention of every head of one query token over a shared latent cache.

    q [B, H, 576] bf16, kv [B, Sk, 576] bf16 (V = kv[..., :512]) → (O [B, H, 512] bf16,
    LSE [B, H] fp32).  Split-KV across ~2 waves of CTAs, merged by an LSE-weighted combine."""
    if q.dim() != 3 or kv.dim() != 3 or q.shape[-1] != MLA_DQK or kv.shape[-1] != MLA_DQK \
            or q.shape[0] != kv.shape[0]:
        raise ShapeError("mla_decode wants q [B,H,576], kv [B,Sk,576]", q=tuple(q.shape),
                         kv=tuple(kv.shape))
    q = q.to(_BF16).contiguous()
    kv = kv.to(_BF16).contiguous()
    B, H, _ = q.shape
    c = rt.MlaDesc()
    c.batch, c.heads, c.seq_k, c.d_qk, c.d_v, c.scale = B, H, kv.shape[1], MLA_DQK, MLA_DV, scale
    c.splits = int(splits)
    o = torch.empty(B, H, MLA_DV, device=q.device, dtype=_BF16)
    lse = torch.empty(B, H, device=q.device, dtype=torch.float32)
    L = rt.lib()
    ws_n = L.af_mla_decode_workspace(c)
    ws = torch.empty(ws_n, device=q.device, dtype=torch.uint8)
    rt.check(L.af_mla_decode(c, q.data_ptr(), kv.data_ptr(), o.data_ptr(), lse.data_ptr(),
                             ws.data_ptr(), ws_n, _stream()), "af_mla_decode")
    return o, lse


def _fused_dims(spec, plan, precision: str) -> bool:
    """Head dims the fused kernels are instantiated for (directly, zero-padded, as 128-wide value
    slices, or as MLA)."""
    d = spec.dims
    if spec.kv_shared:
        return (d.d_qk, d.d_v) == (MLA_DQK, MLA_DV) and d.kv_heads == 1 and precision == "bf16"
    if precision != "bf16":
        return d.d_qk <= 128 and d.d_v <= 128
    dims = (d.d_qk, d.d_v)
    return (dims in _KERNEL_DIMS or max(dims) <= 128 or dims == (128, 256))


def route_parallel(spec, arrays: dict | None = None, precision: str = "bf16"):
    """("fused", ParallelPlan) when the fused kernels lower the variant at these dims (and, for
    the abssum family, the decay mask is its declared fill); otherwise ("generic", GenericPlan)
    — the materialised tier (generic.py) — which raises UnsupportedError for what neither
    lowers."""
    spec = _spec(spec)
    try:
        plan = plan_parallel(spec)
    except UnsupportedError as fused_err:
        try:
            return "generic", generic.plan_generic(spec)
        except UnsupportedError:
            raise fused_err from None
    if not _fused_dims(spec, plan, precision):
        return "generic", generic.plan_generic(spec)
    if plan.family == FAMILY_ABSSUM and arrays is not None and plan.decay_extra in arrays:
        try:
            _check_decay_mask(plan, arrays[plan.decay_extra], arrays[plan.decay_extra].device)
        except UnsupportedError:
            return "generic", generic.plan_generic(spec)
    return "fused", plan


def parallel_forward(spec, arrays: dict, *, precision: str = "bf16", check_nan: bool = False):
    """Forward of the parallel template → ``(O [B,H,Sq,Dv], LSE [B,H,Sq] fp32 or None)``.

    ``precision="bf16"`` runs the tcgen05 kernel (K1) on bf16 inputs (fp32 inputs are rounded);
    ``"fp32"`` runs the exact-FFMA fp32 kernel (cfg1 parity path).  MLA variants (``kv_shared``,
    (Dqk, Dv) = (576, 512), one latent head) run K3: prefill, or the split-KV decode kernel when
    seq_q == 1 and no mask applies.  An ``output_mod`` runs on the full output afterwards
    (af_hook_eval); the LSE is the template's own row statistic."""
    spec = _spec(spec)
    route, plan = route_parallel(spec, arrays, precision)
    if route == "generic":
        o, lse = generic.forward(plan, arrays, _BF16 if precision == "bf16" else torch.float32)
        if check_nan:
            _check_nan(o, "materialised")
        return o, lse
    o, lse = _parallel_forward_core(spec, plan, arrays, precision)
    if "o" in plan.hooks:
        o = _out_mod(plan, o, arrays)
    if check_nan:
        _check_nan(o, "kernel")
    return o, lse


def _parallel_forward_core(spec, plan, arrays: dict, precision: str):
    d0 = spec.dims
    if (spec.kv_shared and precision == "bf16" and (d0.d_qk, d0.d_v) == (MLA_DQK, MLA_DV)
            and d0.seq_q == 1 and not plan.band.causal and plan.band.window is None):
        q = _need(arrays, "q")
        k = _need(arrays, "k")
        _check_shape(q, (d0.batch, d0.heads, 1, MLA_DQK), "q")
        _check_shape(k, (d0.batch, 1, d0.seq_k, MLA_DQK), "k")
        o, lse = mla_decode(q[:, :, 0], k[:, 0], float(plan.scale),
                            int(_tuning(spec).get("splits", 0)))
        return o.unsqueeze(2), lse.unsqueeze(2)
    dtype = _BF16 if precision == "bf16" else torch.float32
    q, k, v, slope = _parallel_inputs(plan, arrays, dtype)
    d = spec.dims
    pad = _padded_dim(spec, precision)
    if pad is not None:
        q, k, v = _pad_last(q, pad), _pad_last(k, pad), _pad_last(v, pad)
    o = _empty("fwd.o", (d.batch, d.heads, d.seq_q, v.shape[-1]), dtype, q.device)
    lse = (_empty("fwd.lse", (d.batch, d.heads, d.seq_q), torch.float32, q.device)
           if plan.has_lse else None)
    # Value dims above the kernel's 128 (softmax-diff's 256) run as 128-wide value slices: the
    # normalised scores P do not depend on V, so each slice is exact (S is recomputed per slice)
    vw = 128 if (precision == "bf16" and v.shape[-1] > 128 and v.shape[-1] % 128 == 0
                 and q.shape[-1] <= 128) else v.shape[-1]
    for c0 in range(0, v.shape[-1], vw):
        vs, os_ = v[..., c0:c0 + vw], o[..., c0:c0 + vw]
        desc = _desc(plan, q, k, vs, os_, slope,
                     rt.AF_DTYPE_BF16 if dtype == _BF16 else rt.AF_DTYPE_F32)
        rt.check(rt.lib().af_parallel_fwd(desc, q.data_ptr(), k.data_ptr(), vs.data_ptr(),
                                          os_.data_ptr(), rt.ptr(lse), _stream()),
                 "af_parallel_fwd")
    if pad is not None:
        o = o[..., : d.d_v].contiguous()
    return o, lse


def run_tiled_parallel(spec, arrays: dict, block_q: int = 64, block_k: int = 64, **kw):
    """Drop-in for ``engine.run_tiled_parallel`` (engine.py:423).  The kernel's own 128x128 tile
    replaces ``block_q``/``block_k`` (the reference pins tiled ≡ naive for any blocking,
    test_engine.py:189-205)."""
    if block_q < 1 or block_k < 1:
        raise InputError("block sizes must be positive", block_q=block_q, block_k=block_k)
    return parallel_forward(spec, arrays, check_nan=True, **kw)[0]


def run_naive_parallel(spec, arrays: dict, **kw):
    return parallel_forward(spec, arrays, check_nan=True, **kw)[0]


def parallel_backward(spec, arrays: dict, o: torch.Tensor, lse, dout: torch.Tensor) -> dict:
    """VJP of ``parallel_forward`` for cotangent ``dout``: ``{"q": dq, "k": dk, "v": dv}`` (bf16;
    dk/dv summed over each GQA group; for ``kv_shared`` the V gradient is folded into dk), plus
    the gradient of every differentiable extra read by a whole-tensor hook (q/k/v mod programs,
    output_mod).  With an ``output_mod`` the template's own output is recomputed (``o`` is the
    modified one) and ``dout`` is pulled back through the mod first."""
    spec = _spec(spec)
    route, plan = route_parallel(spec, arrays)
    if route == "generic":
        return generic.backward(plan, arrays, dout)
    grads_x: dict = {}
    if "o" in plan.hooks:
        o, lse = _parallel_forward_core(spec, plan, arrays, "bf16")
        dout = _out_mod_vjp(plan, o, dout, arrays, grads_x)
    g = _parallel_backward_mapped(spec, plan, arrays, o, lse, dout)
    for name, kind in zip("qkv", _maps(plan)):  # chain the q/k/v mods: dL/dx = dL/df(x) f'(x)
        if kind and name in g:
            g[name] = _mod_vjp(plan, name, _need(arrays, name), g[name], arrays, grads_x)
    for name, t in grads_x.items():
        g[name] = t.reshape(_need(arrays, name).shape).to(torch.float32)
    return g


def _parallel_backward_mapped(spec, plan, arrays: dict, o, lse, dout) -> dict:
    q, k, v, slope = _parallel_inputs(plan, arrays, _BF16)
    d = spec.dims
    pad = _padded_dim(spec, "bf16")
    if pad is not None:
        g = parallel_backward_padded(spec, plan, (q, k, v, slope), o, lse, dout, pad)
        return g
    o = _as(o, _BF16)
    dout = _as(dout, _BF16).contiguous() if dout.stride() != o.stride() else _as(dout, _BF16)
    if dout.stride() != o.stride():
        dout = dout.contiguous()
        o = o.contiguous()
    _check_shape(dout, (d.batch, d.heads, d.seq_q, d.d_v), "dout")
    dq = _empty("bwd.dq", q.shape, q.dtype, q.device)
    dk = _empty("bwd.dk", k.shape, _BF16, k.device)
    if spec.kv_shared:
        # MLA lowering: V aliases K[..., :d_v]; the kernel writes dK + [dV, 0] into dk
        if q.stride() != dq.stride() or k.stride() != dk.stride():
            q, k = q.contiguous(), k.contiguous()
        v = k[..., : d.d_v]
        dv = dk[..., : d.d_v]
    else:
        dv = _empty("bwd.dv", (d.batch, d.kv_heads, d.seq_k, d.d_v), _BF16, k.device)
        # dq/dk/dv are written with the q/k/v strides of the descriptor: use contiguous copies
        if q.stride() != dq.stride() or k.stride() != dk.stride() or v.stride() != dv.stride():
            q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    desc = _desc(plan, q, k, v, o, slope, rt.AF_DTYPE_BF16)
    L = rt.lib()
    ws_n = L.af_parallel_bwd_workspace(desc)
    ws = _empty("bwd.ws", (ws_n,), torch.uint8, q.device)
    if plan.family in (FAMILY_SOFTMAX, FAMILY_ABSSUM) and lse is None:
        raise InputError("softmax / abssum backward needs the forward row statistic")
    rt.check(L.af_parallel_bwd(desc, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                               rt.ptr(lse), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                               dv.data_ptr(), ws.data_ptr(), ws_n, _stream()), "af_parallel_bwd")
    if spec.kv_shared:
        return {"q": dq, "k": dk}
    return {"q": dq, "k": dk, "v": dv}


def parallel_backward_padded(spec, plan, qkvs, o, lse, dout, pad: int) -> dict:
    """Backward on zero-padded head dims (see ``_padded_dim``); gradients sliced back."""
    q, k, v, slope = qkvs
    d = spec.dims
    q, k, v = (_pad_last(t, pad).contiguous() for t in (q, k, v))
    o = _pad_last(_as(o, _BF16), pad).contiguous()
    dout = _pad_last(_as(dout, _BF16), pad).contiguous()
    _check_shape(dout, (d.batch, d.heads, d.seq_q, pad), "dout")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    desc = _desc(plan, q, k, v, o, slope, rt.AF_DTYPE_BF16)
    L = rt.lib()
    ws_n = L.af_parallel_bwd_workspace(desc)
    ws = torch.empty(ws_n, device=q.device, dtype=torch.uint8)
    if plan.family in (FAMILY_SOFTMAX, FAMILY_ABSSUM) and lse is None:
        raise InputError("softmax / abssum backward needs the forward row statistic")
    rt.check(L.af_parallel_bwd(desc, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                               rt.ptr(lse), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                               dv.data_ptr(), ws.data_ptr(), ws_n, _stream()), "af_parallel_bwd")
    return {"q": dq[..., : d.d_qk].contiguous(), "k": dk[..., : d.d_qk].contiguous(),
            "v": dv[..., : d.d_v].contiguous()}


# ───────────────────────────── recurrent template ─────────────────────────────

def _step_tensor(arrays: dict, name: str, d) -> torch.Tensor:
    t = _need(arrays, name)
    if t.dim() != 4 or t.shape[2] != d.seq_k or t.shape[3] != 1:
        raise ShapeError("per-step extra must be [B|1, H|1, seq, 1]", name=name,
                         got=tuple(t.shape))
    return t.to(torch.float32).contiguous()


def _linear_desc(plan: LinearPlan, arrays: dict, q, k, v, o):
    """Descriptor + the fp32 per-step tensors it points to (kept alive by the caller)."""
    d = plan.spec.dims
    c = rt.LinearDesc()
    c.batch, c.heads, c.seq = d.batch, d.heads, d.seq_q
    c.d_k, c.d_v = int(q.shape[-1]), int(v.shape[-1])  # kernel (possibly padded) dims
    c.chunk = 128
    c.decay_hint = int(plan.decay_hint)
    c.q_scale = float(plan.q_scale)
    c.q_stride, c.k_stride, c.v_stride, c.o_stride = (rt.strides4(q), rt.strides4(k),
                                                      rt.strides4(v), rt.strides4(o))
    if plan.decay_const <= 0:
        raise UnsupportedError("per-step decay constant must be positive", value=plan.decay_const)
    c.log_decay_const = math.log(plan.decay_const)
    keep = {}
    if len(plan.decay_factors) > 2:
        raise UnsupportedError("at most two per-step decay factors", n=len(plan.decay_factors))
    c.n_decay_factors = len(plan.decay_factors)
    for f, name in enumerate(plan.decay_factors):
        t = keep.setdefault(name, _step_tensor(arrays, name, d))
        c.decay_factor[f] = t.data_ptr()
        c.decay_factor_stride[f] = rt.step_strides(t)
    if plan.k_gate is not None:
        t = keep.setdefault(plan.k_gate, _step_tensor(arrays, plan.k_gate, d))
        c.key_gate = t.data_ptr()
        c.key_gate_stride = rt.step_strides(t)
    return c, keep


def _check_factors(plan: LinearPlan, arrays: dict) -> None:
    """The chunked kernels evaluate decays in log space: a negative per-step factor has no
    log-space form (the reference's running product handles it, engine.py:597-605)."""
    for name in plan.decay_factors:
        t = _need(arrays, name)
        if bool((t < 0).any().item()):
            raise UnsupportedError("negative per-step decay factor; the chunked kernels need "
                                   "a_t >= 0", extra=name)


def _linear_pad(d) -> tuple[int, int]:
    """Kernel dims of the linear template: 128 or 256 for both the key and the value dim (the
    backward runs the chunked kernel with the value dim in the key role).  Smaller dims run
    zero-padded (zero q/k columns add nothing to q.k or to the state, zero v columns only produce
    sliced-off output columns); the q_mod scale comes from the spec."""
    def up(n):
        return 128 if n <= 128 else (256 if n <= 256 else n)
    return up(d.d_qk), up(d.d_v)


def _linear_qkv(plan: LinearPlan, arrays: dict):
    d = plan.spec.dims
    q, k, v = _need(arrays, "q"), _need(arrays, "k"), _need(arrays, "v")
    _check_shape(q, (d.batch, d.heads, d.seq_q, d.d_qk), "q")
    _check_shape(k, (d.batch, d.heads, d.seq_k, d.d_qk), "k")
    _check_shape(v, (d.batch, d.heads, d.seq_k, d.d_v), "v")
    q, k, v = (_mod(plan, n, t, arrays) for n, t in (("q", q), ("k", k), ("v", v)))
    pk, pv = _linear_pad(d)
    return (_pad_last(_as(q, _BF16), pk), _pad_last(_as(k, _BF16), pk),
            _pad_last(_as(v, _BF16), pv))


def linear_forward(spec, arrays: dict, chunk: int = 128, *, check_nan: bool = False,
                   return_state: bool = False):
    """Chunked linear template forward (K4) → O [B,H,S,Dv] bf16.  The decay factors of h_mod
    and the k_mod gate are applied inside the kernel.  ``return_state=True`` also returns the
    fp32 state after the last token, [B,H,Dk,Dv] (the recurrence's h_S, for ``linear_step``)."""
    spec = _spec(spec)
    plan = plan_linear(spec, chunk)
    q, k, v = _linear_qkv(plan, arrays)
    d = spec.dims
    o = _empty("lin.o", (d.batch, d.heads, d.seq_q, v.shape[-1]), _BF16, q.device)
    state = (torch.empty(d.batch, d.heads, q.shape[-1], v.shape[-1], device=q.device,
                         dtype=torch.float32) if return_state else None)
    desc, _keep = _linear_desc(plan, arrays, q, k, v, o)
    L = rt.lib()
    ws_n = L.af_linear_fwd_workspace(desc)
    ws = _empty("lin.fws", (ws_n,), torch.uint8, q.device)
    rt.check(L.af_linear_fwd(desc, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                             rt.ptr(state), ws.data_ptr(), ws_n, _stream()), "af_linear_fwd")
    if o.shape[-1] != d.d_v:
        o = o[..., : d.d_v].contiguous()
    if "o" in plan.hooks:
        o = _out_mod(plan, o, arrays)
    if check_nan:
        if torch.isnan(o).any().item():
            _check_factors(plan, arrays)
        _check_nan(o, "chunk")
    if return_state:
        return o, state[..., : d.d_qk, : d.d_v].contiguous()
    return o


def linear_step(spec, arrays: dict, state: torch.Tensor) -> torch.Tensor:
    """One generation step of the recurrent template (K4s): ``arrays`` hold ONE new token
    (q/k/v [B,H,1,D], per-step extras [B|1,H|1,1,1]); ``state`` (fp32 [B,H,Dk,Dv], e.g. from
    ``linear_forward(..., return_state=True)``) is advanced in place; returns o_t [B,H,1,Dv].
    The body of engine.run_step_recurrent (engine.py:539-547) for a carried state."""
    spec = _spec(spec)
    d = spec.dims
    if d.seq_q != 1 or d.seq_k != 1:
        raise ShapeError("linear_step takes a one-token spec (seq = 1)", seq=d.seq_q)
    plan = plan_linear(spec)
    q, k, v = _need(arrays, "q"), _need(arrays, "k"), _need(arrays, "v")
    _check_shape(q, (d.batch, d.heads, 1, d.d_qk), "q")
    _check_shape(k, (d.batch, d.heads, 1, d.d_qk), "k")
    _check_shape(v, (d.batch, d.heads, 1, d.d_v), "v")
    q, k, v = (_as(_mod(plan, n, t, arrays), _BF16).contiguous()
               for n, t in (("q", q), ("k", k), ("v", v)))
    if state.dtype != torch.float32 or tuple(state.shape) != (d.batch, d.heads, d.d_qk, d.d_v) \
            or not state.is_contiguous() or not state.is_cuda:
        raise ShapeError("state must be contiguous fp32 [B,H,Dk,Dv] on the GPU",
                         got=tuple(state.shape))
    o = torch.empty(d.batch, d.heads, 1, d.d_v, device=q.device, dtype=_BF16)
    desc, _keep = _linear_desc(plan, arrays, q, k, v, o)
    rt.check(rt.lib().af_linear_step(desc, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                     state.data_ptr(), o.data_ptr(), _stream()), "af_linear_step")
    return _out_mod(plan, o, arrays)


def run_chunk_recurrent(spec, arrays: dict, chunk: int = 64):
    """Drop-in for ``engine.run_chunk_recurrent`` (engine.py:554).  The kernel's own chunk (128)
    replaces ``chunk`` (chunked ≡ stepwise for any chunking, test_engine.py:208-221)."""
    if chunk < 1:
        raise InputError("chunk must be positive", chunk=chunk)
    return linear_forward(spec, arrays, check_nan=True)


def run_step_recurrent(spec, arrays: dict):
    """Drop-in for ``engine.run_step_recurrent`` (engine.py:525)."""
    return linear_forward(spec, arrays, check_nan=True)


def linear_backward(spec, arrays: dict, dout: torch.Tensor, chunk: int = 128) -> dict:
    """VJP of ``linear_forward`` (K5): grads for q, k, v and every differentiable extra that
    enters a_t or k_mod (accumulated in-kernel with the extra's broadcast shape)."""
    spec = _spec(spec)
    plan = plan_linear(spec, chunk)
    d = spec.dims
    _check_shape(dout, (d.batch, d.heads, d.seq_q, d.d_v), "dout")
    hook_grads: dict = {}
    if "o" in plan.hooks:  # pull dout back through output_mod at the template's own output
        o_inner = linear_forward(dataclasses.replace(spec, output_mod=None), arrays, chunk)
        dout = _out_mod_vjp(plan, o_inner, _as(dout, _BF16), arrays, hook_grads)
    q, k, v = (t.contiguous() for t in _linear_qkv(plan, arrays))
    dout = _as(dout, _BF16).contiguous()
    dout = _pad_last(dout, v.shape[-1]).contiguous()
    dq = _empty("lin.dq", q.shape, q.dtype, q.device)
    dk = _empty("lin.dk", k.shape, k.dtype, k.device)
    dv = _empty("lin.dv", v.shape, v.dtype, v.device)
    # dout / dq use the o / q stride slots of the descriptor (all contiguous here)
    desc, keep = _linear_desc(plan, arrays, q, k, v, dout)
    extras = spec.extras_by_name()
    grads_x = {name: torch.zeros(t.shape, device=q.device, dtype=torch.float32)
               for name, t in keep.items() if extras[name].differentiable}
    dfac = (rt.C.c_void_p * 2)()
    for f, name in enumerate(plan.decay_factors):
        if name in grads_x:
            dfac[f] = grads_x[name].data_ptr()
    dgate = grads_x.get(plan.k_gate) if plan.k_gate is not None else None
    L = rt.lib()
    ws_n = L.af_linear_bwd_workspace(desc)
    ws = _empty("lin.ws", (ws_n,), torch.uint8, q.device)
    rt.check(L.af_linear_bwd(desc, q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(),
                             dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                             rt.C.cast(dfac, rt.C.c_void_p), rt.ptr(dgate), ws.data_ptr(), ws_n,
                             _stream()), "af_linear_bwd")
    grads = {"q": dq[..., : d.d_qk], "k": dk[..., : d.d_qk], "v": dv[..., : d.d_v]}
    grads = {n: (t if t.is_contiguous() else t.contiguous()) for n, t in grads.items()}
    for name, kind in zip("qkv", _maps(plan)):  # chain the q/k/v mods
        if kind:
            grads[name] = _mod_vjp(plan, name, _need(arrays, name), grads[name], arrays,
                                   hook_grads)
    for name, g in grads_x.items():
        grads[name] = g.reshape(_need(arrays, name).shape)
    for name, g in hook_grads.items():
        g = g.reshape(_need(arrays, name).shape).to(torch.float32)
        grads[name] = grads[name] + g if name in grads else g
    return grads


# ───────────────────────────── autodiff entry point ─────────────────────────────

def autodiff_grads(spec, arrays: dict, wrt=None, dout: torch.Tensor | None = None) -> dict:
    """Drop-in for ``engine.autodiff_grads`` (engine.py:630): gradients of ``sum(O)`` (or of
    ``<dout, O>`` when ``dout`` is given) with respect to q, k, v and differentiable extras."""
    spec = _spec(spec)
    d = spec.dims
    if spec.pattern is Pattern.PARALLEL:
        o, lse = parallel_forward(spec, arrays)
        g = torch.ones_like(o) if dout is None else dout
        _check_extra_grads(spec, arrays)
        grads = parallel_backward(spec, arrays, o, lse, g)
    else:
        g = torch.ones(d.batch, d.heads, d.seq_q, d.d_v, device=_need(arrays, "q").device,
                       dtype=_BF16) if dout is None else dout
        grads = linear_backward(spec, arrays, g)
    if wrt is None:
        wrt = ["q", "k", "v"] + [e.name for e in spec.extra_inputs if e.differentiable]
    missing = [n for n in wrt if n not in grads]
    if missing:
        raise InputError("cannot differentiate unknown inputs", names=missing)
    return {n: grads[n] for n in wrt}


# ───────────────────────────── bound executable ─────────────────────────────

@dataclass
class BoundKernel:
    """``lowering.bind_executable(assemble_kernel(spec, tile), plan)`` analogue: the lowered plan
    bound to the sm_100a kernels; ``run(arrays)`` executes it (lowering.py:857-860)."""

    spec: AttentionSpec
    plan: object

    def run(self, arrays: dict) -> torch.Tensor:
        if self.spec.pattern is Pattern.PARALLEL:
            return run_tiled_parallel(self.spec, arrays)
        return run_chunk_recurrent(self.spec, arrays)


def bind(spec) -> BoundKernel:
    spec = _spec(spec)
    plan = route_parallel(spec)[1] if spec.pattern is Pattern.PARALLEL else plan_linear(spec)
    return BoundKernel(spec, plan)


# ───────────────────────────── autograd module ─────────────────────────────

class _ParallelFn(torch.autograd.Function):
    """Autograd node of the parallel template.  Extras are positional inputs (names on ctx) so
    autograd sees them.  Extras read by whole-tensor hooks (q/k/v mod programs, output_mod) get
    gradients; a differentiable extra read by the fused score hooks raises at forward time (the
    reference differentiates it, attention.py:542-543; not lowered here)."""

    @staticmethod
    def forward(ctx, spec, names, q, k, v, *extra_t):
        extras = dict(zip(names, extra_t))
        _check_extra_grads(spec, {"q": q, "k": k, "v": v, **extras})
        arrays = {"q": q, "k": k, "v": v, **extras}
        with torch.cuda.device(q.device):
            o, lse = parallel_forward(spec, arrays)
        ctx.spec, ctx.names = spec, names
        ctx.save_for_backward(q, k, v, o, lse if lse is not None else torch.empty(0), *extra_t)
        ctx.has_lse = lse is not None
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse, *extra_t = ctx.saved_tensors
        arrays = {"q": q, "k": k, "v": v, **dict(zip(ctx.names, extra_t))}
        with torch.cuda.device(q.device):
            g = parallel_backward(ctx.spec, arrays, o, lse if ctx.has_lse else None, do)
        # MLA (kv_shared): V aliases K[..., :d_v]; its gradient is folded into dk and the v
        # argument is not read, so it receives none.
        gv = g.get("v")
        gx = [g[n].to(t.dtype) if n in g and ctx.needs_input_grad[5 + i] else None
              for i, (n, t) in enumerate(zip(ctx.names, extra_t))]
        return (None, None, g["q"].to(q.dtype), g["k"].to(k.dtype),
                gv.to(v.dtype) if gv is not None and v is not None else None, *gx)


class AttentionEngine:
    """AttentionEngine-style callable: ``AttentionEngine(spec)(q, k, v, **custom_fwd_inputs)``
    with autograd support (forward K1, backward K2 / linear K4-K5).  Gradients flow to q, k, v
    and, on the linear template, to the differentiable per-step extras (gate / decay)."""

    def __init__(self, spec):
        self.spec = _spec(spec)
        self.plan = bind(self.spec).plan

    def __call__(self, q, k, v, **extras):
        names = tuple(extras)
        tensors = tuple(extras[n] for n in names)
        if self.spec.pattern is Pattern.PARALLEL:
            return _ParallelFn.apply(self.spec, names, q, k, v, *tensors)
        return _LinearFn.apply(self.spec, names, q, k, v, *tensors)


class _LinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, spec, names, q, k, v, *extra_t):
        ctx.spec, ctx.names = spec, names
        ctx.save_for_backward(q, k, v, *extra_t)
        return linear_forward(spec, {"q": q, "k": k, "v": v, **dict(zip(names, extra_t))})

    @staticmethod
    def backward(ctx, do):
        q, k, v, *extra_t = ctx.saved_tensors
        with torch.cuda.device(q.device):
            g = linear_backward(ctx.spec, {"q": q, "k": k, "v": v,
                                           **dict(zip(ctx.names, extra_t))}, do)
        gx = [g[n].to(t.dtype) if n in g and ctx.needs_input_grad[5 + i] else None
              for i, (n, t) in enumerate(zip(ctx.names, extra_t))]
        return None, None, g["q"].to(q.dtype), g["k"].to(k.dtype), g["v"].to(v.dtype), *gx
