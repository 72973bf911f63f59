"""Linear (recurrent) template oracle, float64.  TEST INFRASTRUCTURE ONLY.

``step_forward``   restates engine.run_step_recurrent (engine.py:525-551):
                   h <- h_mod(h) + k_t^T v_t ; o_t = q_t h ; h_0 = 0 ; output_mod after.
``chunk_forward``  restates engine.run_chunk_recurrent (engine.py:554-616) including its
                   running-product decay table (597-605) and state update (606-612).
``chunk_vjp``      gradients of <dO, O> by the chunked reverse scan of SURVEY Appendix A.4
                   (log-space decay, validated there against attention.RecurrenceDef.unroll +
                   graph.backward at S <= 256, which is the reference's unroll cap,
                   attention.py:452).  Hook derivatives (k_mod, q_mod, v_mod, per-step scale)
                   follow the reference adjoint rules through ``hooks.evaluate_dual``.
"""

from __future__ import annotations

import ast
import math

import numpy as np

from .hooks import compile_hook, evaluate, evaluate_dual

_ERR = dict(divide="ignore", invalid="ignore", over="ignore", under="ignore")


def _consts(d) -> dict:
    return {"batch": float(d.batch), "heads": float(d.heads), "seqq": float(d.seq_q),
            "seqk": float(d.seq_k), "dimqk": float(d.d_qk), "dimv": float(d.d_v)}


def scale_source(spec) -> str | None:
    """diagonal_scale (attention.py:332-369) on the oracle's AST: the per-step factor when h_mod
    is ``h * f1 * f2 ...``; '1' for identity; None when it does not factor."""
    if spec.h_mod is None:
        return "1"
    hname = spec.h_mod.input_name or "h"
    tree = compile_hook(spec.h_mod.source)
    factors: list = []

    def flat(n):
        if isinstance(n, ast.BinOp) and isinstance(n.op, ast.Mult):
            flat(n.left)
            flat(n.right)
        else:
            factors.append(n)

    flat(tree)
    hs = [f for f in factors if isinstance(f, ast.Name) and f.id == hname]
    rest = [f for f in factors if not (isinstance(f, ast.Name) and f.id == hname)]
    if len(hs) != 1:
        return None
    for f in rest:
        if any(isinstance(x, ast.Name) and x.id == hname for x in ast.walk(f)):
            return None
    if not rest:
        return "1"
    return " * ".join(f"({ast.unparse(f)})" for f in rest)


def _full(x, shape):
    return np.asarray(x, np.float64) * np.ones(shape)


def _premod(spec, arrays):
    """engine._premod_qkv (engine.py:511-522)."""
    env = {**_consts(spec.dims), **arrays}
    q, k, v = (np.asarray(arrays[n], np.float64) for n in "qkv")
    qm = evaluate(spec.q_mod.source, {**env, "q": q}) if spec.q_mod else q
    km = evaluate(spec.k_mod.source, {**env, "k": k}) if spec.k_mod else k
    vm = evaluate(spec.v_mod.source, {**env, "v": v}) if spec.v_mod else v
    return _full(qm, q.shape), _full(km, k.shape), _full(vm, v.shape)


def per_step_scale(spec, arrays) -> np.ndarray:
    src = scale_source(spec)
    if src is None:
        raise NotImplementedError("h_mod does not factor as h * a_t")
    d = spec.dims
    return _full(evaluate(src, {**_consts(d), **arrays}), (d.batch, d.heads, d.seq_k, 1))


def _output_mod(spec, arrays, out):
    if spec.output_mod is None:
        return out
    return _full(evaluate(spec.output_mod.source, {**_consts(spec.dims), **arrays, "o": out}),
                 out.shape)


def step_forward(spec, arrays: dict) -> np.ndarray:
    """engine.run_step_recurrent (engine.py:525-551)."""
    d = spec.dims
    consts = _consts(d)
    qm, km, vm = _premod(spec, arrays)
    h = np.zeros((d.batch, d.heads, d.d_qk, d.d_v))
    out = np.zeros((d.batch, d.heads, d.seq_q, d.d_v))
    with np.errstate(**_ERR):
        for t in range(d.seq_q):
            env = dict(consts)
            for e in spec.extra_inputs:
                env[e.name] = np.asarray(arrays[e.name], np.float64)[..., t:t + 1, :]
            if spec.h_mod is not None:
                h = _full(evaluate(spec.h_mod.source, {**env, "h": h}), h.shape)
            h = h + np.swapaxes(km[..., t:t + 1, :], -1, -2) @ vm[..., t:t + 1, :]
            out[..., t:t + 1, :] = qm[..., t:t + 1, :] @ h
    return _output_mod(spec, arrays, out)


def chunk_forward(spec, arrays: dict, chunk: int = 64) -> np.ndarray:
    """engine.run_chunk_recurrent (engine.py:554-616), running-product decay table."""
    d = spec.dims
    qm, km, vm = _premod(spec, arrays)
    sc = per_step_scale(spec, arrays)
    b, hh = d.batch, d.heads
    h = np.zeros((b, hh, d.d_qk, d.d_v))
    out = np.zeros((b, hh, d.seq_q, d.d_v))
    with np.errstate(**_ERR):
        for c0 in range(0, d.seq_q, chunk):
            cs = slice(c0, min(c0 + chunk, d.seq_q))
            c = cs.stop - cs.start
            qc, kc, vc, scc = qm[..., cs, :], km[..., cs, :], vm[..., cs, :], sc[..., cs, :]
            dmat = np.zeros((b, hh, c, c))
            dmat[..., 0, 0] = 1.0
            for i in range(1, c):
                dmat[..., i, :i] = dmat[..., i - 1, :i] * scc[..., i, :]
                dmat[..., i, i] = 1.0
            cp = np.ones((b, hh, c, 1))
            cp[..., 0, :] = scc[..., 0, :]
            for i in range(1, c):
                cp[..., i, :] = cp[..., i - 1, :] * scc[..., i, :]
            a = (qc @ np.swapaxes(kc, -1, -2)) * dmat
            out[..., cs, :] = a @ vc + (qc * cp) @ h
            w = np.swapaxes(dmat[..., c - 1:c, :], -1, -2)
            h = cp[..., c - 1, :][..., None] * h + np.swapaxes(kc * w, -1, -2) @ vc
    return _output_mod(spec, arrays, out)


def chunk_vjp(spec, arrays: dict, dout: np.ndarray, chunk: int = 64) -> dict[str, np.ndarray]:
    """Gradients of <dout, O> w.r.t. q, k, v and the differentiable extras."""
    d = spec.dims
    consts = _consts(d)
    qm, km, vm = _premod(spec, arrays)
    sc = per_step_scale(spec, arrays)
    dout = np.asarray(dout, np.float64)
    if spec.output_mod is not None:
        o_inner = chunk_forward(_no_output_mod(spec), arrays, chunk)
        _, dm = evaluate_dual(spec.output_mod.source, {**consts, **arrays, "o": o_inner}, "o")
        dout = dout * dm
    b, hh, S = d.batch, d.heads, d.seq_q
    with np.errstate(**_ERR):
        loga = np.log(sc[..., 0])                       # [b, h, S]
        # forward pass storing chunk input states
        starts = list(range(0, S, chunk))
        h_in = []
        h = np.zeros((b, hh, d.d_qk, d.d_v))
        for c0 in starts:
            cs = slice(c0, min(c0 + chunk, S))
            L = np.cumsum(loga[..., cs], axis=-1)
            w = np.exp(L[..., -1:] - L)[..., None]
            h_in.append(h)
            h = np.exp(L[..., -1])[..., None, None] * h + \
                np.swapaxes(km[..., cs, :] * w, -1, -2) @ vm[..., cs, :]
        dqm, dkm, dvm = np.zeros_like(qm), np.zeros_like(km), np.zeros_like(vm)
        dloga = np.zeros_like(loga)
        dH = np.zeros((b, hh, d.d_qk, d.d_v))
        for ci in reversed(range(len(starts))):
            c0 = starts[ci]
            cs = slice(c0, min(c0 + chunk, S))
            n = cs.stop - cs.start
            L = np.cumsum(loga[..., cs], axis=-1)       # [b,h,n]
            idx = np.arange(n)
            tril = idx[:, None] >= idx[None, :]
            D = np.where(tril, np.exp(L[..., :, None] - L[..., None, :]), 0.0)
            cp = np.exp(L)[..., None]                   # [b,h,n,1]
            wv = np.exp(L[..., -1:] - L)[..., None]     # [b,h,n,1]
            Q, K, V, dO, Hin = qm[..., cs, :], km[..., cs, :], vm[..., cs, :], dout[..., cs, :], \
                h_in[ci]
            A = Q @ np.swapaxes(K, -1, -2)
            G = dO @ np.swapaxes(V, -1, -2)
            GD = G * D
            dqm[..., cs, :] = GD @ K + cp * (dO @ np.swapaxes(Hin, -1, -2))
            dkm[..., cs, :] = np.swapaxes(GD, -1, -2) @ Q + wv * (V @ np.swapaxes(dH, -1, -2))
            dvm[..., cs, :] = np.swapaxes(A * D, -1, -2) @ dO + wv * (K @ dH)
            AGD = A * GD                                  # [b,h,i,u]
            # intra: sum_{i>=j} sum_{u<j} AGD[i,u]
            rowpre = np.cumsum(AGD, axis=-1)               # sum_{u<=t}
            intra = np.zeros_like(L)
            for j in range(n):
                if j > 0:
                    intra[..., j] = rowpre[..., j:, j - 1].sum(-1)
            inter_out = np.flip(np.cumsum(np.flip(
                cp[..., 0] * np.sum(dO * (Q @ Hin), -1), -1), -1), -1)
            carry = np.exp(L[..., -1]) * np.sum(dH * Hin, axis=(-1, -2))
            upd = wv[..., 0] * np.sum(K * (V @ np.swapaxes(dH, -1, -2)), -1)  # per u
            upd_pre = np.concatenate([np.zeros_like(upd[..., :1]), np.cumsum(upd, -1)[..., :-1]],
                                     -1)
            dloga[..., cs] = intra + inter_out + carry[..., None] + upd_pre
            dH = np.exp(L[..., -1])[..., None, None] * dH + np.swapaxes(Q * cp, -1, -2) @ dO
    # chain through the hooks
    env = {**consts, **arrays}
    q, k, v = (np.asarray(arrays[n], np.float64) for n in "qkv")
    grads = {
        "q": dqm * _full(evaluate_dual(spec.q_mod.source, {**env, "q": q}, "q")[1], q.shape)
        if spec.q_mod else dqm,
        "k": dkm * _full(evaluate_dual(spec.k_mod.source, {**env, "k": k}, "k")[1], k.shape)
        if spec.k_mod else dkm,
        "v": dvm * _full(evaluate_dual(spec.v_mod.source, {**env, "v": v}, "v")[1], v.shape)
        if spec.v_mod else dvm,
    }
    src = scale_source(spec)
    for e in spec.extra_inputs:
        if not e.differentiable:
            continue
        x = np.asarray(arrays[e.name], np.float64)
        full = (b, hh, S, 1)
        g = np.zeros(full)
        a_val, a_d = evaluate_dual(src, {**env}, e.name)
        g += dloga[..., None] * _full(a_d, full) / _full(a_val, full)
        for nm, fn, dm in (("q", spec.q_mod, dqm), ("k", spec.k_mod, dkm), ("v", spec.v_mod, dvm)):
            if fn is not None and e.name in {n.id for n in ast.walk(compile_hook(fn.source))
                                             if isinstance(n, ast.Name)}:
                src_arr = np.asarray(arrays[nm], np.float64)
                _, dd = evaluate_dual(fn.source, {**env, nm: src_arr}, e.name)
                g += np.sum(dm * _full(dd, dm.shape), -1, keepdims=True)
        axes = tuple(i for i, (have, want) in enumerate(zip(full, x.shape))
                     if want == 1 and have != 1)
        grads[e.name] = g.sum(axis=axes, keepdims=True) if axes else g
    return grads


def _no_output_mod(spec):
    fields = {f: getattr(spec, f) for f in spec.__dataclass_fields__}
    fields["output_mod"] = None
    return spec.__class__(**fields)


_ = math
