"""Generate golden fixtures from the reference implementation itself.

Runs ONLY in the build container, where the reference (attnforge, read-only) is importable from
/root/reference/pkg/src.  Writes tests/golden/<case>.npz with the variant (as variant-file JSON),
the seed, the reference-generated inputs and the reference's outputs:

  o_tiled   engine.run_tiled_parallel / run_chunk_recurrent
  o_naive   engine.run_naive_parallel / run_step_recurrent
  lse       run_tiled_parallel on the same variant with the softmax online protocol and epilogue
            ``acc * 0 + m + log(l)``; broadcast column 0 kept
  dout, g_* engine.autodiff_grads of the variant with ``output_mod = o * g`` and extra ``g = dout``
             — i.e. the VJP for an arbitrary cotangent

Usage:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import os
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from attnforge import attention as A  # noqa: E402
from attnforge import engine as E  # noqa: E402
from attnforge import variantfile as VF  # noqa: E402

OUT = Path(__file__).resolve().parent


def to_doc(spec) -> dict:
    d = spec.dims
    doc = {"name": spec.name, "pattern": spec.pattern.value,
           "dims": {"batch": d.batch, "heads": d.heads, "seq_q": d.seq_q, "seq_k": d.seq_k,
                    "dqk": d.d_qk, "dv": d.d_v}}
    for f in ("q_mod", "k_mod", "v_mod", "output_mod", "h_mod"):
        fn = getattr(spec, f)
        if fn is not None:
            doc[f] = fn.source
    plain = [m for m in spec.score_mods if not m.ismask]
    masks = [m for m in spec.score_mods if m.ismask]
    assert len(plain) <= 1 and (not plain or spec.score_mods[0] is plain[0])
    if plain:
        doc["score_mod"] = plain[0].source
    if masks:
        doc["masks"] = [{"expr": m.source, "ismask": True} for m in masks]
    rn = spec.rownorm
    if isinstance(rn, A.DirectRowNorm):
        doc["rownorm"] = {"direct": rn.body.source}
    elif isinstance(rn, A.OnlineRowNorm):
        doc["rownorm"] = {"online": {"rowscales": list(rn.rowscales),
                                     "prologue": {n: f.source for n, f in rn.prologue},
                                     "fwd": {n: f.source for n, f in rn.fwd},
                                     "epilogue": rn.epilogue.source}}
        if rn.direct is not None:
            doc["rownorm_direct"] = rn.direct.body.source  # informational
    if spec.extra_inputs:
        doc["extras"] = [{"name": e.name, "shape": list(e.shape), "fill": e.fill,
                          "fill_params": dict(e.fill_params),
                          "differentiable": e.differentiable} for e in spec.extra_inputs]
    return doc


def lse_spec(spec):
    rn = A.online(rowscales=["m", "l"], prologue={"m": "-inf", "l": "0"},
                  fwd={"m_new": "max(m, reduceMax(s))",
                       "r": "where(m_new == -inf, 1, exp(m - m_new))",
                       "p": "where(m_new == -inf, 0, exp(s - m_new))",
                       "l": "r * l + reduceSum(p)", "m": "m_new", "scores": "p",
                       "rescale": "r"},
                  epilogue="acc * 0 + m + log(l)")
    return replace(spec, rownorm=rn)


def vjp_spec(spec):
    tok = "seq_q" if spec.pattern is A.Pattern.PARALLEL else "seq_k"
    g = A.ExtraInput("g", ("batch", "heads", tok, "d_v"), "uniform", differentiable=False)
    return replace(spec, output_mod=A.mod("o * g", "o"), extra_inputs=spec.extra_inputs + (g,))


def case(name: str, spec, seed: int, *, lse: bool = False, grads: bool = True,
         chunk: int = 16) -> None:
    inst = E.generate(spec, seed)
    arrays = inst.arrays
    rec = {"doc": json.dumps(to_doc(spec)), "seed": seed}
    for k, v in arrays.items():
        rec[f"in_{k}"] = v
    if spec.pattern is A.Pattern.PARALLEL:
        rec["o_tiled"] = E.run_tiled_parallel(spec, arrays, 16, 16)
        rec["o_naive"] = E.run_naive_parallel(spec, arrays)
        if lse:
            rec["lse"] = E.run_tiled_parallel(lse_spec(spec), arrays, 16, 16)[..., 0]
    else:
        rec["o_tiled"] = E.run_chunk_recurrent(spec, arrays, chunk)
        rec["o_naive"] = E.run_step_recurrent(spec, arrays)
    if grads:
        vs = vjp_spec(spec)
        rng = np.random.Generator(np.random.Philox(key=(seed << 32) + 777))
        dout = rng.uniform(-1, 1, size=rec["o_tiled"].shape)
        va = dict(arrays)
        va["g"] = dout
        wrt = ["q", "k", "v"] + [e.name for e in spec.extra_inputs if e.differentiable]
        gr = E.autodiff_grads(vs, va, wrt)
        rec["dout"] = dout
        for k, v in gr.items():
            rec[f"g_{k}"] = v
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print(f"{name}: {', '.join(sorted(rec))}")


def main() -> None:
    tiny = dict(heads=1, seq_q=8, seq_k=8, d_qk=4, d_v=4)
    for b in A.BUILTIN_NAMES:
        kw = dict(tiny)
        if b in A.RECURRENT_BUILTINS:
            kw.pop("seq_k")
        sp = A.builtin(b, **kw)
        case(f"tiny_{b}", sp, 0, lse=b.startswith("softmax"), chunk=3)
        if sp.pattern is A.Pattern.PARALLEL:
            case(f"tiny_causal_{b}", A.with_causal_mask(sp), 1, lse=b.startswith("softmax"))
    # medium parallel shapes
    sp = A.with_causal_mask(A.builtin("softmax", batch=1, heads=2, seq_q=96, seq_k=96, d_qk=32,
                                      d_v=32))
    case("softmax_causal_s96_d32", sp, 3, lse=True)
    sp = A.builtin("softmax", batch=2, heads=1, seq_q=40, seq_k=72, d_qk=16, d_v=16)
    case("softmax_ragged_q40_k72", sp, 4, lse=True)
    sp = A.with_causal_mask(A.builtin("softmax-deepseek", batch=1, heads=2, seq=48, d_qk=24,
                                      d_v=16))
    case("deepseek_causal_s48", sp, 5, lse=True)
    # cfg3-style variant: sigmoid + relative position + causal + sliding window
    doc = {"name": "sigmoid-relpos-swa", "pattern": "parallel",
           "dims": {"batch": 1, "heads": 2, "seq_q": 80, "seq_k": 80, "dqk": 16, "dv": 16},
           "q_mod": "q / sqrt(dimqk)",
           "score_mod": "sigmoid(s - slope * (qidx - kidx) - log(seqk))",
           "masks": [{"expr": "s * where(kidx <= qidx, 1, 0)", "ismask": True},
                     {"expr": "s * where(qidx - kidx < 24, 1, 0)", "ismask": True}],
           "extras": [{"name": "slope", "shape": [1, "heads", 1, 1], "fill": "constant_decay",
                       "fill_params": {"gamma": [2 ** (-8 * (h + 1) / 2) for h in range(2)]},
                       "differentiable": False}]}
    case("sigmoid_relpos_swa", VF.spec_from_dict(doc), 6)
    sp = A.with_causal_mask(A.builtin("relu", batch=1, heads=2, seq=64, d_qk=16, d_v=16))
    case("relu_causal_s64", sp, 7)
    # packaged variant files
    vdir = Path(REF) / "attnforge" / "data" / "variants"
    for f in sorted(vdir.glob("*.json")):
        sp = VF.load_variant(str(f))
        d = sp.dims
        sp = replace(sp, dims=A.Dims(1, 2, min(d.seq_q, 48), min(d.seq_k, 48), 16, 16))
        case(f"variant_{f.stem}", sp, 8, lse=f.stem == "capped-softmax")
    # recurrent, longer than one chunk
    case("retention_s64", A.builtin("retention-recurrent", batch=1, heads=2, seq=64, d_qk=16,
                                    d_v=16), 9)
    case("gated_retention_s64", A.builtin("gated-retention", batch=1, heads=2, seq=64, d_qk=16,
                                          d_v=8), 10)
    case("mamba2_s80", A.builtin("mamba2-ssm", batch=2, heads=2, seq=80, d_qk=16, d_v=8), 11)


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
