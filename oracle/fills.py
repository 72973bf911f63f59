"""Deterministic problem instances — restates attnforge ``engine.generate`` (engine.py:326-388).
TEST INFRASTRUCTURE ONLY.

Each tensor draws from its own Philox stream keyed ``(seed << 32) + role`` (roles q=0, k=1, v=2,
extras 3.. in declaration order; index grids consume no stream), so the oracle regenerates the
reference's inputs bit-exactly without importing the reference.
"""

from __future__ import annotations

import numpy as np

_MASK64 = (1 << 64) - 1


def philox_key(seed: int, role: int) -> int:
    return ((seed & _MASK64) << 32) + role  # engine.py:326-327


def _rng(seed: int, role: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=philox_key(seed, role)))


def _extent(dims, tok) -> int:
    if tok == 1:
        return 1
    return {"batch": dims.batch, "heads": dims.heads, "seq_q": dims.seq_q, "seq_k": dims.seq_k,
            "d_qk": dims.d_qk, "d_v": dims.d_v}[tok]


def fill(name: str, shape_tokens, fill_kind: str, params: dict, dims, seed: int, role: int,
         heads_for_kv: int | None = None):
    """engine._fill (engine.py:334-359)."""
    ext = tuple(_extent(dims, t) for t in shape_tokens)
    if heads_for_kv is not None:  # GQA extension: K/V carry heads_kv heads
        ext = (ext[0], heads_for_kv) + ext[2:]
    if fill_kind == "uniform":
        return _rng(seed, role).uniform(-1.0, 1.0, size=ext)
    if fill_kind == "unit":
        return 0.5 + 0.45 * _rng(seed, role).uniform(-1.0, 1.0, size=ext)
    if fill_kind == "constant_decay":
        g = np.asarray(params["gamma"], dtype=np.float64)
        return np.broadcast_to(g[None, :, None, None], ext).copy()
    if fill_kind == "causal_decay_mask":
        g = np.asarray(params["gamma"], dtype=np.float64)
        delta = (np.arange(dims.seq_q)[:, None] - np.arange(dims.seq_k)[None, :]).astype(float)
        out = np.zeros((1, dims.heads, dims.seq_q, dims.seq_k))
        with np.errstate(all="ignore"):
            for h in range(dims.heads):
                out[0, h] = np.where(delta >= 0, g[h] ** np.maximum(delta, 0.0), 0.0)
        return out
    if fill_kind == "index_q":
        return np.arange(dims.seq_q, dtype=np.float64).reshape(1, 1, -1, 1)
    if fill_kind == "index_k":
        return np.arange(dims.seq_k, dtype=np.float64).reshape(1, 1, 1, -1)
    raise ValueError(f"unknown fill policy {fill_kind!r} for {name}")


def input_descriptors(spec):
    """(name, shape tokens, fill, params, differentiable) like AttentionSpec.input_descriptors
    (attention.py:219-233)."""
    out = [("q", ("batch", "heads", "seq_q", "d_qk"), "uniform", {}, True),
           ("k", ("batch", "heads", "seq_k", "d_qk"), "uniform", {}, True),
           ("v", ("batch", "heads", "seq_k", "d_v"), "uniform", {}, True)]
    for e in spec.extra_inputs:
        out.append((e.name, tuple(e.shape), e.fill, dict(e.fill_params), e.differentiable))
    names = set()
    from .hooks import free_names
    for m in spec.score_mods:
        names |= free_names(m.source)
    if names & {"qidx", "kidx"}:
        out.append(("qidx", (1, 1, "seq_q", 1), "index_q", {}, False))
        out.append(("kidx", (1, 1, 1, "seq_k"), "index_k", {}, False))
    return out


def generate(spec, seed: int) -> dict[str, np.ndarray]:
    """engine.generate (engine.py:369-388).  With the GQA extension (``dims.heads_kv``) K/V are
    drawn with heads_kv heads from the same streams."""
    arrays: dict[str, np.ndarray] = {}
    role = 0
    hkv = getattr(spec.dims, "heads_kv", None)
    for name, shape, kind, params, _ in input_descriptors(spec):
        if name in ("q", "k", "v"):
            r = {"q": 0, "k": 1, "v": 2}[name]
        elif name in ("qidx", "kidx"):
            r = 0
        else:
            r = 3 + role
            role += 1
        arrays[name] = fill(name, shape, kind, params, spec.dims, seed, r,
                            heads_for_kv=hkv if name in ("k", "v") and hkv else None)
    return arrays
