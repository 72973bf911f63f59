"""Parallel template oracle (float64).  TEST INFRASTRUCTURE ONLY.

``tiled_forward``   restates engine.run_tiled_parallel (engine.py:423-505): per query block the
                    online prologue initialises row scales (469-472); per key block the scores are
                    produced (474), score/mask mods applied in order (478-480), the fwd
                    assignments run (483-484) and ``acc = acc*rescale + p@V`` (487); epilogue
                    (496-499), output_mod on the full output (502-504), NaN raises (391-395).
``naive_forward``   restates run_naive_parallel / build_parallel (engine.py:401-406,
                    attention.py:389-449): dense scores, direct rownorm (or the whole-row online
                    protocol when no direct form is declared).
``lse_rows``        log-sum-exp of the final score rows — what the reference's own online
                    epilogue ``acc*0 + m + log(l)`` returns.
``streamed_vjp``    the same forward + VJP streamed over query-row blocks (full-length slices at
                    O(block * S) memory); ``keycols_softmax_vjp`` dK/dV of sampled key rows summed
                    over every query head given the forward's row statistics.
``parallel_vjp``    gradients of <dO, O> in closed form, equal to what
                    attention.derive_backward + graph.backward produce with the ``o * g``
                    cotangent trick; elementwise hook derivatives use the
                    reference adjoint rules (graph.py:481-569) via ``hooks.evaluate_dual``.

Extensions (documented gaps of the reference): GQA (``dims.heads_kv``: K/V expanded
with repeat-interleave, dK/dV group-summed) and MLA (``kv_shared``: V = K[..., :d_v]).
Contractions use numpy matmul in float64; the reference's pinned ascending accumulation order
(engine.py:44-80) differs from it by ~1e-16 relative, far below every tolerance used here.
"""

from __future__ import annotations

import math

import numpy as np

from .hooks import evaluate, evaluate_dual, row_max, row_sum

_ERR = dict(divide="ignore", invalid="ignore", over="ignore", under="ignore")


def _consts(dims) -> dict:
    return {"batch": float(dims.batch), "heads": float(dims.heads), "seqq": float(dims.seq_q),
            "seqk": float(dims.seq_k), "dimqk": float(dims.d_qk), "dimv": float(dims.d_v)}


def _group(spec) -> int:
    hkv = getattr(spec.dims, "heads_kv", None)
    return 1 if hkv is None else spec.dims.heads // hkv


def _expand(x: np.ndarray, g: int) -> np.ndarray:
    return x if g == 1 else np.repeat(x, g, axis=1)


def _inputs(spec, arrays):
    """Modified q/k/v at full head count (engine.py:445-452)."""
    env = {**_consts(spec.dims), **arrays}
    g = _group(spec)
    q = np.asarray(arrays["q"], np.float64)
    k = _expand(np.asarray(arrays["k"], np.float64), g)
    if getattr(spec, "kv_shared", False):
        v = k[..., : spec.dims.d_v]
    else:
        v = _expand(np.asarray(arrays["v"], np.float64), g)
    qm = evaluate(spec.q_mod.source, {**env, "q": q}) if spec.q_mod else q
    km = evaluate(spec.k_mod.source, {**env, "k": k}) if spec.k_mod else k
    vm = evaluate(spec.v_mod.source, {**env, "v": v}) if spec.v_mod else v
    ones = np.ones
    return (np.asarray(qm, np.float64) * ones(q.shape), np.asarray(km, np.float64) * ones(k.shape),
            np.asarray(vm, np.float64) * ones(v.shape))


def _index_env(spec, qs=slice(None), ks=slice(None)) -> dict:
    d = spec.dims
    return {"qidx": np.arange(d.seq_q, dtype=np.float64)[qs].reshape(1, 1, -1, 1),
            "kidx": np.arange(d.seq_k, dtype=np.float64)[ks].reshape(1, 1, 1, -1)}


def _extra_view(spec, arr, shape_tokens, qs, ks):
    idx = [slice(None)] * 4
    for ax, tok in enumerate(shape_tokens):
        if tok == "seq_q" and arr.shape[ax] > 1:
            idx[ax] = qs
        elif tok == "seq_k" and arr.shape[ax] > 1:
            idx[ax] = ks
    return arr[tuple(idx)]


def _rownorm_kind(rn):
    if rn is None:
        return None
    return "online" if hasattr(rn, "rowscales") else "direct"


def _check(out, what):
    if np.isnan(out).any():
        raise FloatingPointError(f"output contains NaN ({what})")
    return out


def tiled_forward(spec, arrays: dict, block_q: int = 64, block_k: int = 64) -> np.ndarray:
    """engine.run_tiled_parallel (engine.py:423-505)."""
    d = spec.dims
    consts = _consts(d)
    qm, km, vm = _inputs(spec, arrays)
    rn = spec.rownorm
    kind = _rownorm_kind(rn)
    if kind == "direct":
        block_k = d.seq_k  # engine.py:457-458
    extras = {e.name: e for e in spec.extra_inputs}
    b, h = d.batch, d.heads
    out = np.zeros((b, h, d.seq_q, d.d_v))
    with np.errstate(**_ERR):
        for q0 in range(0, d.seq_q, block_q):
            qs = slice(q0, min(q0 + block_q, d.seq_q))
            bq = qs.stop - qs.start
            acc = np.zeros((b, h, bq, d.d_v))
            scales = {}
            if kind == "online":
                for name, fn in rn.prologue:
                    scales[name] = np.full((b, h, bq, 1), evaluate(fn.source, dict(consts)))
            for k0 in range(0, d.seq_k, block_k):
                ks = slice(k0, min(k0 + block_k, d.seq_k))
                s = np.matmul(qm[..., qs, :], np.swapaxes(km[..., ks, :], -1, -2))
                env = {**consts, **_index_env(spec, qs, ks)}
                for name, e in extras.items():
                    env[name] = _extra_view(spec, np.asarray(arrays[name], np.float64), e.shape,
                                            qs, ks)
                for m in spec.score_mods:
                    env["s"] = s
                    s = np.asarray(evaluate(m.source, env), np.float64) * np.ones(s.shape)
                if kind == "online":
                    fenv = {**consts, **scales, "s": s}
                    for name, fn in rn.fwd:
                        fenv[name] = evaluate(fn.source, fenv)
                    p = np.asarray(fenv["scores"], np.float64) * np.ones(s.shape)
                    acc = acc * fenv["rescale"] + p @ vm[..., ks, :]
                    scales = {n: np.asarray(fenv[n]) * np.ones((b, h, bq, 1))
                              for n in rn.rowscales}
                elif kind == "direct":
                    s = np.asarray(evaluate(rn.body.source, {**consts, "s": s}), np.float64)
                    acc = acc + s @ vm[..., ks, :]
                else:
                    acc = acc + s @ vm[..., ks, :]
            if kind == "online":
                acc = np.asarray(evaluate(rn.epilogue.source, {**consts, **scales, "acc": acc}),
                                 np.float64) * np.ones(acc.shape)
            out[..., qs, :] = acc
    if spec.output_mod is not None:
        out = np.asarray(evaluate(spec.output_mod.source,
                                  {**consts, **arrays, "o": out}), np.float64)
    return _check(out, "tiled")


def final_scores(spec, arrays: dict):
    """Dense scores after every score/mask mod, with d(score)/d(raw score)
    (elementwise chain rule through the mods)."""
    d = spec.dims
    qm, km, vm = _inputs(spec, arrays)
    s_raw = np.matmul(qm, np.swapaxes(km, -1, -2))
    env = {**_consts(d), **_index_env(spec)}
    for e in spec.extra_inputs:
        env[e.name] = np.asarray(arrays[e.name], np.float64)
    z, dz = s_raw, np.ones_like(s_raw)
    for m in spec.score_mods:
        z, dz = evaluate_dual(m.source, {**env, "s": z}, "s", seed=dz)
        z = np.asarray(z, np.float64) * np.ones(s_raw.shape)
        dz = np.asarray(dz, np.float64) * np.ones(s_raw.shape)
    return qm, km, vm, s_raw, z, dz


def _softmax(z):
    with np.errstate(**_ERR):
        m = row_max(z)
        ok = np.isfinite(m)
        e = np.where(ok, np.exp(z - np.where(ok, m, 0.0)), 0.0)
        den = row_sum(e)
        return np.where(den == 0, 0.0, e / np.where(den == 0, 1.0, den))


def _classify(spec) -> str:
    """Which closed form the rownorm follows (numeric fingerprint on random rows)."""
    rn = spec.rownorm
    if rn is None:
        return "none"
    consts = _consts(spec.dims)
    rng = np.random.default_rng(99)
    z = rng.uniform(-4, 4, size=(1, 1, 5, 12))
    z[0, 0, 1, :5] = -np.inf
    z[0, 0, 2, :] = -np.inf
    zf = np.where(np.isfinite(z), z, 0.0)
    with np.errstate(**_ERR):
        if _rownorm_kind(rn) == "direct":
            got = np.asarray(evaluate(rn.body.source, {**consts, "s": z}), np.float64)
            gotf = np.asarray(evaluate(rn.body.source, {**consts, "s": zf}), np.float64)
        else:
            got = _whole_row_online(rn, consts, z)
            gotf = _whole_row_online(rn, consts, zf)
    if np.allclose(got, _softmax(z), atol=1e-12, equal_nan=False):
        return "softmax"
    a = np.sum(np.abs(zf), -1, keepdims=True)
    if np.allclose(gotf, zf / np.clip(a, 1, None), atol=1e-12):
        return "abssum"
    raise NotImplementedError("oracle VJP has no closed form for this rownorm")


def _whole_row_online(rn, consts, s):
    b, h, r, n = s.shape
    scales = {nm: np.full((b, h, r, 1), evaluate(fn.source, dict(consts)))
              for nm, fn in rn.prologue}
    fenv = {**consts, **scales, "s": s}
    for nm, fn in rn.fwd:
        fenv[nm] = evaluate(fn.source, fenv)
    p = np.asarray(fenv["scores"], np.float64) * np.ones(s.shape)
    sc = {nm: np.asarray(fenv[nm]) * np.ones((b, h, r, 1)) for nm in rn.rowscales}
    return np.asarray(evaluate(rn.epilogue.source, {**consts, **sc, "acc": p}),
                      np.float64) * np.ones(s.shape)


def naive_forward(spec, arrays: dict) -> np.ndarray:
    """run_naive_parallel (engine.py:401-406) via build_parallel semantics."""
    consts = _consts(spec.dims)
    qm, km, vm, s_raw, z, dz = final_scores(spec, arrays)
    rn = spec.rownorm
    with np.errstate(**_ERR):
        if rn is None:
            out = z @ vm
        elif _rownorm_kind(rn) == "direct" or rn.direct is not None:
            body = rn.body if _rownorm_kind(rn) == "direct" else rn.direct.body
            out = np.asarray(evaluate(body.source, {**consts, "s": z}), np.float64) @ vm
        else:
            out = _whole_row_online_out(rn, consts, z, vm)
    if spec.output_mod is not None:
        out = np.asarray(evaluate(spec.output_mod.source, {**consts, **arrays, "o": out}))
    return _check(out, "naive")


def _whole_row_online_out(rn, consts, s, vm):
    b, h, r, n = s.shape
    scales = {nm: np.full((b, h, r, 1), evaluate(fn.source, dict(consts)))
              for nm, fn in rn.prologue}
    fenv = {**consts, **scales, "s": s}
    for nm, fn in rn.fwd:
        fenv[nm] = evaluate(fn.source, fenv)
    acc = (np.asarray(fenv["scores"], np.float64) * np.ones(s.shape)) @ vm
    sc = {nm: np.asarray(fenv[nm]) * np.ones((b, h, r, 1)) for nm in rn.rowscales}
    return np.asarray(evaluate(rn.epilogue.source, {**consts, **sc, "acc": acc}), np.float64)


def lse_rows(spec, arrays: dict) -> np.ndarray:
    """[B, H, Sq] log-sum-exp of the final scores (−inf for fully-masked rows)."""
    _, _, _, _, z, _ = final_scores(spec, arrays)
    with np.errstate(**_ERR):
        m = row_max(z)
        ok = np.isfinite(m)
        l = row_sum(np.where(ok, np.exp(z - np.where(ok, m, 0.0)), 0.0))
        lse = np.where(l == 0, -np.inf, np.where(ok, m, 0.0) + np.log(np.where(l == 0, 1.0, l)))
    return lse[..., 0]


def forward_with_lse(spec, arrays: dict):
    o = tiled_forward(spec, arrays)
    lse = lse_rows(spec, arrays) if _classify(spec) == "softmax" else None
    return o, lse


def parallel_vjp(spec, arrays: dict, dout: np.ndarray) -> dict[str, np.ndarray]:
    """Gradients of <dout, O> w.r.t. q, k, v."""
    d = spec.dims
    consts = _consts(d)
    kind = _classify(spec)
    qm, km, vm, s_raw, z, dz = final_scores(spec, arrays)
    dout = np.asarray(dout, np.float64)
    with np.errstate(**_ERR):
        if spec.output_mod is not None:
            o_inner = naive_forward(spec.__class__(**{**_fields(spec), "output_mod": None}),
                                    arrays) if hasattr(spec, "__dataclass_fields__") else None
            _, dmod = evaluate_dual(spec.output_mod.source, {**consts, **arrays, "o": o_inner},
                                    "o")
            dout = dout * dmod
        if kind == "softmax":
            p = _softmax(z)
            o = p @ vm
            dp = dout @ np.swapaxes(vm, -1, -2)
            delta = row_sum(dout * o)
            dzz = p * (dp - delta)
            pv = p
        elif kind == "none":
            dzz = dout @ np.swapaxes(vm, -1, -2)
            pv = z
        else:  # abssum-clamp rownorm (attention.py:575-586; graph.py:528-557)
            a = row_sum(np.abs(z))
            c = np.clip(a, 1.0, None)
            o = (z @ vm) / c
            dp = dout @ np.swapaxes(vm, -1, -2)
            sign = np.where(z >= 0, 1.0, -1.0)
            dzz = dp / c - (a >= 1.0) * sign * row_sum(dout * o) / c
            pv = z / c
        ds = dzz * dz
        ds = np.where(np.isfinite(ds), ds, 0.0)
        dqm = ds @ km
        dkm = np.swapaxes(ds, -1, -2) @ qm
        dvm = np.swapaxes(pv, -1, -2) @ dout
    env = {**consts, **arrays}
    g = _group(spec)
    q = np.asarray(arrays["q"], np.float64)
    k = _expand(np.asarray(arrays["k"], np.float64), g)
    dq = dqm * (evaluate_dual(spec.q_mod.source, {**env, "q": q}, "q")[1] if spec.q_mod else 1.0)
    dk = dkm * (evaluate_dual(spec.k_mod.source, {**env, "k": k}, "k")[1] if spec.k_mod else 1.0)
    if getattr(spec, "kv_shared", False):
        v = k[..., : d.d_v]
    else:
        v = _expand(np.asarray(arrays["v"], np.float64), g)
    dv = dvm * (evaluate_dual(spec.v_mod.source, {**env, "v": v}, "v")[1] if spec.v_mod else 1.0)
    dq = np.asarray(dq) * np.ones(q.shape)
    dk = np.asarray(dk) * np.ones(k.shape)
    dv = np.asarray(dv) * np.ones(v.shape)
    if g > 1:
        b, h = d.batch, d.heads
        dk = dk.reshape(b, h // g, g, d.seq_k, -1).sum(2)
        dv = dv.reshape(b, h // g, g, d.seq_k, -1).sum(2)
    if getattr(spec, "kv_shared", False):
        dk = dk.copy()
        dk[..., : d.d_v] += dv
        return {"q": dq, "k": dk}
    return {"q": dq, "k": dk, "v": dv}


def _fields(spec) -> dict:
    return {f: getattr(spec, f) for f in spec.__dataclass_fields__}


_ = math


def sampled_forward(spec, arrays: dict, rows) -> tuple[np.ndarray, np.ndarray | None]:
    """Dense forward restricted to query rows ``rows`` (absolute indices, so index-grid masks
    stay correct) — for checking full-size kernel outputs on a sample.  Returns (O rows
    [B,H,len(rows),Dv], LSE rows or None)."""
    rows = np.asarray(rows)
    d = spec.dims
    consts = _consts(d)
    qm, km, vm = _inputs(spec, arrays)
    qm = qm[..., rows, :]
    s = np.matmul(qm, np.swapaxes(km, -1, -2))
    env = {**consts, "qidx": rows.astype(np.float64).reshape(1, 1, -1, 1),
           "kidx": np.arange(d.seq_k, dtype=np.float64).reshape(1, 1, 1, -1)}
    for e in spec.extra_inputs:
        x = np.asarray(arrays[e.name], np.float64)
        if e.shape[2] == "seq_q" and x.shape[2] > 1:
            x = x[:, :, rows]
        env[e.name] = x
    with np.errstate(**_ERR):
        for m in spec.score_mods:
            s = np.asarray(evaluate(m.source, {**env, "s": s}), np.float64) * np.ones(s.shape)
        kind = _classify(spec)
        if kind == "softmax":
            p = _softmax(s)
            m_ = row_max(s)
            ok = np.isfinite(m_)
            l = row_sum(np.where(ok, np.exp(s - np.where(ok, m_, 0.0)), 0.0))
            lse = np.where(l == 0, -np.inf, np.where(ok, m_, 0) + np.log(np.where(l == 0, 1, l)))
            return p @ vm, lse[..., 0]
        if kind == "none":
            return s @ vm, None
        a = row_sum(np.abs(s))
        return (s @ vm) / np.clip(a, 1.0, None), None


def _chain_mods(spec, arrays, dqm, dkm, dvm):
    """Chain the q/k/v mods (elementwise) and fold GQA groups / MLA's aliased V, as in
    ``parallel_vjp``."""
    d = spec.dims
    env = {**_consts(d), **arrays}
    g = _group(spec)
    q = np.asarray(arrays["q"], np.float64)
    k = _expand(np.asarray(arrays["k"], np.float64), g)
    v = k[..., : d.d_v] if getattr(spec, "kv_shared", False) else \
        _expand(np.asarray(arrays["v"], np.float64), g)
    dq = dqm * (evaluate_dual(spec.q_mod.source, {**env, "q": q}, "q")[1] if spec.q_mod else 1.0)
    dk = dkm * (evaluate_dual(spec.k_mod.source, {**env, "k": k}, "k")[1] if spec.k_mod else 1.0)
    dv = dvm * (evaluate_dual(spec.v_mod.source, {**env, "v": v}, "v")[1] if spec.v_mod else 1.0)
    dq, dk, dv = (np.asarray(x) * np.ones(y.shape) for x, y in ((dq, q), (dk, k), (dv, v)))
    if g > 1:
        b, h = dk.shape[0], d.heads
        dk = dk.reshape(b, h // g, g, d.seq_k, -1).sum(2)
        dv = dv.reshape(b, h // g, g, d.seq_k, -1).sum(2)
    if getattr(spec, "kv_shared", False):
        dk = dk.copy()
        dk[..., : d.d_v] += dv
        return {"q": dq, "k": dk}
    return {"q": dq, "k": dk, "v": dv}


def _block_scores(spec, env, qm_blk, km, rows, cols):
    """Final scores z and dz/ds of query rows ``rows`` against key columns ``cols`` (absolute
    indices, so index-grid masks stay exact)."""
    s = qm_blk @ np.swapaxes(km, -1, -2)
    env = {**env, "qidx": np.asarray(rows, np.float64).reshape(1, 1, -1, 1),
           "kidx": np.asarray(cols, np.float64).reshape(1, 1, 1, -1)}
    z, dz = s, np.ones_like(s)
    for m in spec.score_mods:
        z, dz = evaluate_dual(m.source, {**env, "s": z}, "s", seed=dz)
        z = np.asarray(z, np.float64) * np.ones(s.shape)
        dz = np.asarray(dz, np.float64) * np.ones(s.shape)
    return z, dz


def _extras_env(spec, arrays, rows, cols):
    env = {}
    for e in spec.extra_inputs:
        x = np.asarray(arrays[e.name], np.float64)
        idx = [slice(None)] * 4
        for ax, tok in enumerate(e.shape):
            if tok == "seq_q" and x.shape[ax] > 1:
                idx[ax] = np.asarray(rows)
            elif tok == "seq_k" and x.shape[ax] > 1:
                idx[ax] = np.asarray(cols)
        env[e.name] = x[tuple(idx)]
    return env


def streamed_vjp(spec, arrays: dict, dout: np.ndarray, block: int = 512) -> dict:
    """Forward and VJP of the softmax / elementwise families streamed over query-row
    blocks, one head at a time, so a full-length slice (S = 8192) needs O(block * S) memory
    instead of O(S^2): the same closed forms as ``parallel_vjp``, exact in float64.
    Returns {"o", "lse" (softmax) , "q", "k", "v"} for the given arrays (any batch / heads)."""
    d = spec.dims
    kind = _classify(spec)
    if kind not in ("softmax", "none"):
        raise NotImplementedError("streamed_vjp covers the softmax and elementwise families")
    qm, km, vm = _inputs(spec, arrays)
    dout = np.asarray(dout, np.float64)
    B, H, S = qm.shape[0], qm.shape[1], d.seq_q
    consts = _consts(d)
    o = np.zeros(qm.shape[:-1] + (vm.shape[-1],))
    lse = np.zeros(qm.shape[:-1]) if kind == "softmax" else None
    dqm, dkm, dvm = np.zeros_like(qm), np.zeros_like(km), np.zeros_like(vm)
    cols = np.arange(d.seq_k)
    with np.errstate(**_ERR):
        for b in range(B):
            for h in range(H):
                for r0 in range(0, S, block):
                    rows = np.arange(r0, min(S, r0 + block))
                    env = {**consts, **_extras_env(spec, arrays, rows, cols)}
                    for k_, x in list(env.items()):
                        if isinstance(x, np.ndarray) and x.ndim == 4:
                            env[k_] = x[min(b, x.shape[0] - 1): min(b, x.shape[0] - 1) + 1,
                                        min(h, x.shape[1] - 1): min(h, x.shape[1] - 1) + 1]
                    qb = qm[b:b + 1, h:h + 1, rows]
                    z, dz = _block_scores(spec, env, qb, km[b:b + 1, h:h + 1], rows, cols)
                    z, dz = z[0, 0], dz[0, 0]
                    vb, kb, dob = vm[b, h], km[b, h], dout[b, h, rows]
                    dp = dob @ vb.T
                    if kind == "softmax":
                        m = np.max(z, -1, keepdims=True)
                        ok = np.isfinite(m)
                        e = np.where(ok, np.exp(z - np.where(ok, m, 0.0)), 0.0)
                        den = np.sum(e, -1, keepdims=True)
                        p = np.where(den == 0, 0.0, e / np.where(den == 0, 1.0, den))
                        lse[b, h, rows] = np.where(den[:, 0] == 0, -np.inf,
                                                   np.where(ok, m, 0.0)[:, 0] + np.log(
                                                       np.where(den == 0, 1.0, den))[:, 0])
                        ob = p @ vb
                        dzz = p * (dp - np.sum(dob * ob, -1, keepdims=True))
                        pv = p
                    else:
                        ob = z @ vb
                        dzz, pv = dp, z
                    o[b, h, rows] = ob
                    ds = dzz * dz
                    ds = np.where(np.isfinite(ds), ds, 0.0)
                    dqm[b, h, rows] = ds @ kb
                    dkm[b, h] += ds.T @ qm[b, h, rows]
                    dvm[b, h] += pv.T @ dob
    g = _chain_mods(spec, arrays, dqm, dkm, dvm)
    g["o"] = o
    if lse is not None:
        g["lse"] = lse
    return g


def keycols_softmax_vjp(spec, arrays: dict, dout: np.ndarray, o: np.ndarray, lse: np.ndarray,
                        key_cols) -> dict:
    """dK (and dV) of the key rows ``key_cols`` only, summed over every query head, for the
    softmax family — given the forward's row statistics (O and LSE, the backward kernel's own
    inputs, each checked against the oracle separately).  Cost O(S * |key_cols|) per head:
    the MLA latent-cache gradient summed over all 128 heads at S = 4096 in seconds.
    Returns {"k": [B, Hkv, |J|, Dqk], "v": [B, Hkv, |J|, Dv]} (MLA: V folded into k)."""
    d = spec.dims
    qm, km, vm = _inputs(spec, arrays)
    J = np.asarray(key_cols)
    dout, o, lse = (np.asarray(x, np.float64) for x in (dout, o, lse))
    consts = _consts(d)
    dkmJ = np.zeros(km.shape[:2] + (len(J), km.shape[-1]))
    dvmJ = np.zeros(vm.shape[:2] + (len(J), vm.shape[-1]))
    rows = np.arange(d.seq_q)
    with np.errstate(**_ERR):
        for b in range(qm.shape[0]):
            for h in range(qm.shape[1]):
                env = {**consts, **_extras_env(spec, arrays, rows, J)}
                z, dz = _block_scores(spec, env, qm[b:b + 1, h:h + 1], km[b:b + 1, h:h + 1, J],
                                      rows, J)
                z, dz = z[0, 0], dz[0, 0]
                lr = lse[b, h][:, None]
                p = np.where(np.isfinite(lr), np.exp(z - np.where(np.isfinite(lr), lr, 0.0)), 0.0)
                dp = dout[b, h] @ vm[b, h, J].T
                delta = np.sum(dout[b, h] * o[b, h], -1, keepdims=True)
                ds = p * (dp - delta) * dz
                ds = np.where(np.isfinite(ds), ds, 0.0)
                dkmJ[b, h] = ds.T @ qm[b, h]
                dvmJ[b, h] = p.T @ dout[b, h]
    g = _group(spec)
    # chain the k / v mods on the selected rows (constant-scale mods in every config here)
    env = {**consts, **arrays}
    k = _expand(np.asarray(arrays["k"], np.float64), g)[..., J, :]
    dk = dkmJ * (evaluate_dual(spec.k_mod.source, {**env, "k": k}, "k")[1] if spec.k_mod else 1.0)
    dv = dvmJ
    if g > 1:
        Bq = dk.shape[0]
        dk = dk.reshape(Bq, d.heads // g, g, len(J), -1).sum(2)
        dv = dv.reshape(Bq, d.heads // g, g, len(J), -1).sum(2)
    if getattr(spec, "kv_shared", False):
        dk = np.asarray(dk, np.float64).copy()
        dk[..., : d.d_v] += dv
        return {"k": dk}
    return {"k": dk, "v": dv}
