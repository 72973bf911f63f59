"""Materialised tier of the parallel template: attnforge ``engine.run_naive_parallel`` /
``build_parallel`` (engine.py:401-406, attention.py:389-449) on the GPU, for variants the fused
kernels (K1/K2/K3) do not lower.

The fused kernels classify each hook into a register epilogue (``plan.py``).  Variants outside
those families — score hooks that read arbitrary materialised extras through the reference's
``_block_view`` semantics (engine.py:413-420, 476-477), softmax with score mods other than a
soft-cap, head dims without a fused instantiation (e.g. retention-parallel's own 256 / 512,
attention.py:682), differentiable extras read by score hooks — run here instead, with the dense
[B, H, Sq, Sk] score tensor materialised exactly as the reference's naive executor does:

  Qm, Km, Vm   the q/k/v mods (a compile-time scale, or a hook program, af_hook_eval)
  S = Qm Km^T  plain fp32 GEMM (cuBLAS through torch.matmul)
  z            every score / mask mod composed into one hook program over the score grid
               (operands: s, the spec's extras broadcast by their strides; qidx / kidx are the
               element's coordinates), with dz/ds from the program's dual number
  P, stat      the recognised rownorm (af_rownorm_fwd: softmax -> LSE, abssum-clamp -> row
               abs-sum, none)
  O = P Vm     plain fp32 GEMM; output_mod as a hook program
  VJP          af_rownorm_bwd + the same GEMMs; gradients of extras read by the score hooks
               are the program's derivative w.r.t. that operand, summed over its broadcast axes
               (graph.py SUM_TO, 575-578).

Memory is O(B·H·Sq·Sk) like the reference's naive executor; calls above ``MAX_BYTES`` raise.
Row normalisations other than softmax / abssum-clamp / none (generic ``online_func`` forms)
raise ``UnsupportedError``.  There is no CPU path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import hooklang as H
from . import hookvm
from . import runtime as rt
from .errors import ShapeError, UnsupportedError
from .plan import FM_NONE, _direct_is_softmax, _feature_map, _np_eval, _substitute, \
    is_online_abssum, is_online_softmax
from .spec import AttentionSpec, DirectRowNorm, OnlineRowNorm, Pattern

MAX_BYTES = 48 << 30  # materialised score scratch per call


@dataclass
class GenericPlan:
    spec: AttentionSpec
    kind: int                               # rt.AF_ROWNORM_*
    score: hookvm.CompiledHook | None       # composed score / mask mods over "s"
    scale: dict = field(default_factory=dict)   # var -> compile-time scalar of a scalar mod
    hooks: dict = field(default_factory=dict)   # var -> CompiledHook ("q"/"k"/"v" mods, "o")

    @property
    def has_stat(self) -> bool:
        return self.kind != rt.AF_ROWNORM_NONE


def _direct_is_abssum(rn: DirectRowNorm, consts) -> bool:
    rng = np.random.default_rng(11)
    s = rng.uniform(-0.2, 0.2, size=(4, 12))
    s[1] *= 0.01
    s[3] *= 10.0
    try:
        got = np.asarray(_np_eval(rn.body.expr, {**consts, "s": s}), float)
    except Exception:  # noqa: BLE001
        return False
    return bool(np.allclose(got, s / np.clip(np.abs(s).sum(-1, keepdims=True), 1, None),
                            atol=1e-12))


def rownorm_kind(spec: AttentionSpec) -> int:
    consts = spec.dims.const_env()
    rn = spec.rownorm
    if rn is None:
        return rt.AF_ROWNORM_NONE
    if isinstance(rn, OnlineRowNorm):
        if is_online_softmax(rn, consts):
            return rt.AF_ROWNORM_SOFTMAX
        if is_online_abssum(rn, consts):
            return rt.AF_ROWNORM_ABSSUM
        # run_tiled_parallel follows the online protocol (engine.py:481-489), not its `direct`
        # twin: an unrecognised online form is not lowered even when a direct body exists
    elif isinstance(rn, DirectRowNorm):
        if _direct_is_softmax(rn, consts):
            return rt.AF_ROWNORM_SOFTMAX
        if _direct_is_abssum(rn, consts):
            return rt.AF_ROWNORM_ABSSUM
    raise UnsupportedError("row normalisation is neither softmax, abssum-clamp nor absent; "
                           "generic online_func forms are not lowered", variant=spec.name)


def plan_generic(spec: AttentionSpec) -> GenericPlan:
    if spec.pattern is not Pattern.PARALLEL:
        raise UnsupportedError("the materialised tier runs the parallel template only")
    spec.validate()
    consts = spec.dims.const_env()
    kind = rownorm_kind(spec)
    extras = [e.name for e in spec.extra_inputs]
    score = None
    if spec.score_mods:
        expr = H.Name("s")
        for m in spec.score_mods:
            expr = _substitute(m.expr, "s", expr)
        score = hookvm.compile_hook(expr, ["s"] + extras, consts,
                                    index_names={"qidx": 2, "kidx": 3})
    scale, hooks = {}, {}
    for var in "qkv":
        fn = getattr(spec, f"{var}_mod")
        kind_m, sc = _feature_map(fn, var, consts)
        if kind_m == FM_NONE:
            scale[var] = sc
        else:  # any non-scalar mod runs as a program (fp32 out)
            hooks[var] = hookvm.compile_hook(fn, [var] + extras, consts)
    if spec.output_mod is not None:
        hooks["o"] = hookvm.compile_hook(spec.output_mod, ["o"] + extras, consts)
    return GenericPlan(spec, kind, score, scale, hooks)


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _extras(spec, arrays) -> dict:
    return {e.name: arrays[e.name] for e in spec.extra_inputs if e.name in arrays}


def _modded(gp: GenericPlan, var: str, x: torch.Tensor, arrays) -> torch.Tensor:
    if var in gp.hooks:
        return hookvm.run_hook(gp.hooks[var], x.shape, {**_extras(gp.spec, arrays), var: x},
                               out_dtype=torch.float32)[0]
    return x.float() * gp.scale.get(var, 1.0)


def _inputs(gp: GenericPlan, arrays):
    spec, d = gp.spec, gp.spec.dims
    q, k = arrays["q"], arrays["k"]
    if tuple(q.shape) != (d.batch, d.heads, d.seq_q, d.d_qk) or \
            tuple(k.shape) != (d.batch, d.kv_heads, d.seq_k, d.d_qk):
        raise ShapeError("q / k shape mismatch", q=tuple(q.shape), k=tuple(k.shape))
    v = k[..., : d.d_v] if spec.kv_shared else arrays["v"]
    if tuple(v.shape) != (d.batch, d.kv_heads, d.seq_k, d.d_v):
        raise ShapeError("v shape mismatch", v=tuple(v.shape))
    g = d.heads // d.kv_heads
    qm, km, vm = (_modded(gp, n, t, arrays) for n, t in (("q", q), ("k", k), ("v", v)))
    if g > 1:
        km, vm = km.repeat_interleave(g, dim=1), vm.repeat_interleave(g, dim=1)
    return qm, km, vm


def _check_budget(d) -> None:
    need = 5 * d.batch * d.heads * d.seq_q * d.seq_k * 4
    if need > MAX_BYTES:
        raise UnsupportedError("the materialised tier would need more score scratch than its "
                               "budget", bytes=need, budget=MAX_BYTES)


def _scores(gp: GenericPlan, arrays, qm, km, want_dz: bool):
    s = torch.matmul(qm, km.transpose(-1, -2))
    if gp.score is None:
        return s, None
    tensors = {**_extras(gp.spec, arrays), "s": s}
    return hookvm.run_hook(gp.score, s.shape, tensors, out_dtype=torch.float32, value=True,
                           wrt="s" if want_dz else None)


def _rownorm(gp: GenericPlan, z: torch.Tensor):
    d = gp.spec.dims
    rows = d.batch * d.heads * d.seq_q
    p = torch.empty_like(z)
    stat = torch.empty(d.batch, d.heads, d.seq_q, device=z.device, dtype=torch.float32) \
        if gp.has_stat else None
    rt.check(rt.lib().af_rownorm_fwd(gp.kind, z.data_ptr(), p.data_ptr(), rt.ptr(stat), rows,
                                     d.seq_k, _stream(z.device)), "af_rownorm_fwd")
    return p, stat


def forward(gp: GenericPlan, arrays: dict, out_dtype=torch.bfloat16):
    """(O [B, H, Sq, Dv], stat [B, H, Sq] or None): LSE for softmax (the fused kernels'
    statistic), the row abs-sum for abssum."""
    d = gp.spec.dims
    _check_budget(d)
    qm, km, vm = _inputs(gp, arrays)
    z, _ = _scores(gp, arrays, qm, km, False)
    p, stat = _rownorm(gp, z)
    del z
    o = torch.matmul(p, vm)
    if "o" in gp.hooks:
        o = hookvm.run_hook(gp.hooks["o"], o.shape, {**_extras(gp.spec, arrays), "o": o},
                            out_dtype=torch.float32)[0]
    return o.to(out_dtype), stat


def _rowdot(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    shape = tuple(a.shape)
    out = torch.empty(shape[:3], device=a.device, dtype=torch.float32)
    oa, ta = hookvm._operand(a, shape, "a")
    ob, tb = hookvm._operand(b, shape, "b")
    shp = (C.c_int32 * 4)(*shape)
    rt.check(rt.lib().af_rowdot(C.addressof(oa), C.addressof(ob), C.addressof(shp),
                                out.data_ptr(), _stream(a.device)), "af_rowdot")
    del ta, tb
    return out


def backward(gp: GenericPlan, arrays: dict, dout: torch.Tensor) -> dict:
    """VJP of ``forward`` for cotangent ``dout``: q, k, v (GQA group-summed; MLA's V folded into
    k) and every differentiable extra read by any hook (score, q/k/v mods, output_mod)."""
    spec, d = gp.spec, gp.spec.dims
    _check_budget(d)
    ext = _extras(spec, arrays)
    grads_x: dict = {}

    def add_x(name, t):
        t = hookvm.sum_to(t, tuple(ext[name].shape))
        grads_x[name] = t if name not in grads_x else grads_x[name] + t

    def hook_x(key, shape, tensors, seed):
        for e in spec.extra_inputs:
            if e.differentiable and gp.hooks[key].uses(e.name):
                add_x(e.name, hookvm.run_hook(gp.hooks[key], shape, tensors, value=False,
                                              wrt=e.name, seed=seed)[1])

    qm, km, vm = _inputs(gp, arrays)
    z, dzds = _scores(gp, arrays, qm, km, True)
    p, stat = _rownorm(gp, z)
    o = torch.matmul(p, vm)
    dout = dout.float()
    if "o" in gp.hooks:
        tensors = {**ext, "o": o}
        _, dout_in = hookvm.run_hook(gp.hooks["o"], o.shape, tensors, value=False, wrt="o",
                                     seed=dout)
        hook_x("o", o.shape, tensors, dout)
        dout = dout_in
    dp = torch.matmul(dout, vm.transpose(-1, -2))
    rowdot = _rowdot(dout, o) if gp.kind != rt.AF_ROWNORM_NONE else None
    gz = torch.empty_like(z)
    rows = d.batch * d.heads * d.seq_q
    rt.check(rt.lib().af_rownorm_bwd(gp.kind, z.data_ptr(), p.data_ptr(), dp.data_ptr(),
                                     rt.ptr(rowdot), rt.ptr(stat), gz.data_ptr(), rows, d.seq_k,
                                     _stream(z.device)), "af_rownorm_bwd")
    del dp
    if gp.score is not None:
        tensors = {**ext, "s": torch.matmul(qm, km.transpose(-1, -2))}
        for e in spec.extra_inputs:
            if e.differentiable and gp.score.uses(e.name):
                add_x(e.name, hookvm.run_hook(gp.score, z.shape, tensors, value=False,
                                              wrt=e.name, seed=gz)[1])
        ds = gz * dzds
    else:
        ds = gz
    ds = torch.where(torch.isfinite(ds), ds, torch.zeros((), device=ds.device))
    dqm = torch.matmul(ds, km)
    dkm = torch.matmul(ds.transpose(-1, -2), qm)
    dvm = torch.matmul(p.transpose(-1, -2), dout)
    del ds, p, z, gz
    q, k = arrays["q"], arrays["k"]
    v = k[..., : d.d_v] if spec.kv_shared else arrays["v"]
    g = d.heads // d.kv_heads
    if g > 1:
        dkm = dkm.reshape(d.batch, d.kv_heads, g, d.seq_k, -1).sum(2)
        dvm = dvm.reshape(d.batch, d.kv_heads, g, d.seq_k, -1).sum(2)
    out = {}
    for var, x, gm in (("q", q, dqm), ("k", k, dkm), ("v", v, dvm)):
        if var in gp.hooks:
            tensors = {**ext, var: x}
            out[var] = hookvm.run_hook(gp.hooks[var], x.shape, tensors, value=False, wrt=var,
                                       seed=gm)[1]
            hook_x(var, x.shape, tensors, gm)
        else:
            out[var] = gm * gp.scale.get(var, 1.0)
    res = {"q": out["q"].to(torch.bfloat16), "k": out["k"], "v": out["v"]}
    if spec.kv_shared:
        kk = res["k"].clone()
        kk[..., : d.d_v] += res.pop("v")
        res["k"] = kk
    res = {n: t.to(torch.bfloat16) for n, t in res.items()}
    for n, t in grads_x.items():
        res[n] = t.reshape(arrays[n].shape).to(torch.float32)
    return res
