"""The BASELINE.json workloads as attention specs, shared by bench.py and the tests.

Each builder returns the spec the reference would be handed for that config — a builtin (plus
``with_causal_mask``) or the variant file of SURVEY §8c(4) — with this package's two extensions
where the config needs them: ``Dims.heads_kv`` (Llama-3 GQA) and ``kv_shared`` (DeepSeek-V2 MLA,
V = K[..., :512]).  Keyword overrides shrink a config for parity tests and CPU samples.
"""

from __future__ import annotations

from dataclasses import replace

from .spec import AttentionSpec, builtin, spec_from_dict, with_causal_mask


def sigmoid_relpos_swa(batch: int = 8, heads: int = 16, seq: int = 4096, d: int = 128,
                       window: int = 1024, heads_kv: int | None = None) -> AttentionSpec:
    """cfg3: sigmoid scores with a per-head relative-position slope, causal + sliding window,
    expressed exactly as the reference variant of SURVEY §8c(4)."""
    doc = {"name": "sigmoid-relpos-swa", "pattern": "parallel",
           "dims": {"batch": batch, "heads": heads, "seq_q": seq, "seq_k": seq, "dqk": d,
                    "dv": d},
           "q_mod": "q / sqrt(dimqk)",
           "score_mod": "sigmoid(s - slope * (qidx - kidx) - log(seqk))",
           "masks": [{"expr": "s * where(kidx <= qidx, 1, 0)", "ismask": True},
                     {"expr": f"s * where(qidx - kidx < {window}, 1, 0)", "ismask": True}],
           "extras": [{"name": "slope", "shape": [1, "heads", 1, 1], "fill": "constant_decay",
                       "fill_params": {"gamma": [2 ** (-8 * (i + 1) / heads)
                                                 for i in range(heads)]},
                       "differentiable": False}]}
    if heads_kv is not None:
        doc["dims"]["heads_kv"] = heads_kv
    return spec_from_dict(doc)


def mla(batch: int, heads: int, seq_q: int, seq_k: int, causal: bool) -> AttentionSpec:
    """DeepSeek-V2 MLA in the absorbed (latent) form: one shared KV head of width 576 whose first
    512 columns are V."""
    sp = builtin("softmax", batch=batch, heads=heads, heads_kv=1, seq_q=seq_q, seq_k=seq_k,
                 d_qk=576, d_v=512)
    sp = replace(sp, kv_shared=True)
    return with_causal_mask(sp) if causal else sp


def cfg1(**kw) -> AttentionSpec:
    a = dict(batch=1, heads=4, seq=512, d=64) | kw
    return with_causal_mask(builtin("softmax", batch=a["batch"], heads=a["heads"], seq=a["seq"],
                                    d_qk=a["d"], d_v=a["d"]))


def cfg2(**kw) -> AttentionSpec:
    a = dict(batch=8, heads=32, heads_kv=8, seq=8192, d=128) | kw
    return with_causal_mask(builtin("softmax", batch=a["batch"], heads=a["heads"],
                                    heads_kv=a["heads_kv"], seq=a["seq"], d_qk=a["d"],
                                    d_v=a["d"]))


def cfg3(**kw) -> AttentionSpec:
    return sigmoid_relpos_swa(**(dict(batch=8, heads=16, seq=4096, d=128, window=1024) | kw))


def cfg4a(**kw) -> AttentionSpec:
    a = dict(batch=1, heads=128, seq=4096) | kw
    return mla(a["batch"], a["heads"], a["seq"], a["seq"], causal=True)


def cfg4b(**kw) -> AttentionSpec:
    a = dict(batch=16, heads=128, seq_k=32768) | kw
    return mla(a["batch"], a["heads"], 1, a["seq_k"], causal=False)


def cfg5a(**kw) -> AttentionSpec:
    a = dict(batch=4, heads=16, seq=8192, d=256) | kw
    return builtin("retention-recurrent", batch=a["batch"], heads=a["heads"], seq=a["seq"],
                   d_qk=a["d"], d_v=a["d"])


def cfg5b(**kw) -> AttentionSpec:
    a = dict(batch=4, heads=32, seq=8192, d=128) | kw
    return builtin("mamba2-ssm", batch=a["batch"], heads=a["heads"], seq=a["seq"], d_qk=a["d"],
                   d_v=a["d"])


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4a": cfg4a, "cfg4b": cfg4b,
           "cfg5a": cfg5a, "cfg5b": cfg5b}


def unmasked_pairs(spec: AttentionSpec) -> int:
    """P = kept (i, j) pairs per (b, h) under the band mask the planner derives."""
    from .plan import plan_parallel
    d = spec.dims
    band = plan_parallel(spec).band
    total = 0
    for i in range(d.seq_q):
        hi = d.seq_k
        if band.upper is not None:
            hi = min(hi, i + band.upper + 1)
        lo = 0
        if band.window is not None:
            lo = max(0, i - band.window + 1)
        total += max(0, hi - lo)
    return total
