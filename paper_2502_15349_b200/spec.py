"""Attention variant specifications — the drop-in construction API.

Same public surface and semantics as the reference (attnforge ``attention.py``):
``Dims``, ``ExtraInput``, ``ModificationFn`` / ``mod``, ``DirectRowNorm``, ``OnlineRowNorm`` /
``online``, ``AttentionSpec`` (+ ``validate``, ``input_descriptors``), ``diagonal_scale``,
``builtin``, ``causal_mask`` / ``with_causal_mask`` and the variant-file loaders
(``variantfile.py``).  AttentionEngine's hook names map onto the fields as follows
(SURVEY §0): ``custom_fwd_inputs`` → ``extra_inputs``; ``score_mod`` / ``mask_mod`` →
``score_mods`` (masks carry ``ismask=True``); ``online_func`` → ``OnlineRowNorm``;
``feature_map`` → ``q_mod``/``k_mod``/``v_mod``; decay hooks → ``h_mod``.

Two extensions the reference lacks (SURVEY §0 "Gaps"), both defaulting to reference behaviour:
``Dims.heads_kv`` (GQA/MQA: K/V carry fewer heads, query head h reads KV head h // group) and
``AttentionSpec.kv_shared`` (MLA: V is the first ``d_v`` columns of K).

``from_reference`` converts an ``attnforge.AttentionSpec`` (duck-typed, no import) so callers can
hand the reference's own objects to this backend.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field, replace
from enum import Enum

from . import hooklang
from .errors import InputError, SchemaError, UnknownVariantError, UnsupportedError, ForgeError

RESERVED_NAMES = {
    "q", "k", "v", "s", "o", "h", "acc", "scores", "rescale", "qidx", "kidx", "inf",
    "batch", "heads", "seqq", "seqk", "dimqk", "dimv",
}


class Pattern(Enum):
    PARALLEL = "parallel"
    RECURRENT = "recurrent"


@dataclass(frozen=True, slots=True)
class Dims:
    batch: int
    heads: int
    seq_q: int
    seq_k: int
    d_qk: int
    d_v: int
    heads_kv: int | None = None  # GQA/MQA extension; None = heads

    def __post_init__(self):
        for name in ("batch", "heads", "seq_q", "seq_k", "d_qk", "d_v"):
            if getattr(self, name) < 1:
                raise InputError(f"dims.{name} must be >= 1", value=getattr(self, name))
        if self.heads_kv is not None and (self.heads_kv < 1 or self.heads % self.heads_kv):
            raise InputError("dims.heads_kv must divide heads", heads=self.heads,
                             heads_kv=self.heads_kv)

    @property
    def kv_heads(self) -> int:
        return self.heads if self.heads_kv is None else self.heads_kv

    def const_env(self) -> dict[str, float]:
        return {"batch": float(self.batch), "heads": float(self.heads),
                "seqq": float(self.seq_q), "seqk": float(self.seq_k),
                "dimqk": float(self.d_qk), "dimv": float(self.d_v)}

    def extent(self, token) -> int:
        if token == 1:
            return 1
        return {"batch": self.batch, "heads": self.heads, "seq_q": self.seq_q,
                "seq_k": self.seq_k, "d_qk": self.d_qk, "d_v": self.d_v}[token]


_SHAPE_TOKENS = ("batch", "heads", "seq_q", "seq_k", "d_qk", "d_v")
FILLS = ("uniform", "unit", "constant_decay", "causal_decay_mask", "index_q", "index_k")


@dataclass(frozen=True, slots=True)
class ExtraInput:
    """A named auxiliary tensor (AttentionEngine ``custom_fwd_inputs``; attention.py:89-121)."""

    name: str
    shape: tuple = ("batch", "heads", "seq_k", 1)
    fill: str = "uniform"
    fill_params: dict = field(default_factory=dict)
    differentiable: bool = True

    def resolve_shape(self, dims: Dims) -> tuple[int, ...]:
        if len(self.shape) != 4:
            raise InputError("extra shapes have rank 4", extra=self.name)
        out = []
        for tok in self.shape:
            if tok != 1 and tok not in _SHAPE_TOKENS:
                raise InputError("bad extra shape token", token=tok, extra=self.name)
            out.append(dims.extent(tok))
        return tuple(out)


@dataclass(frozen=True)
class ModificationFn:
    """One hook fragment over a designated input name (attention.py:124-143)."""

    source: str
    input_name: str | None = None
    ismask: bool = False
    allow_reduce: bool = False
    expr: object = None

    def __post_init__(self):
        if self.expr is None:
            object.__setattr__(self, "expr", hooklang.parse(self.source))

    def free_names(self) -> set[str]:
        return hooklang.free_names(self.expr)


def mod(source: str, input_name: str, *, ismask: bool = False) -> ModificationFn:
    return ModificationFn(source, input_name, ismask=ismask)


@dataclass(frozen=True)
class DirectRowNorm:
    body: ModificationFn

    @classmethod
    def from_source(cls, source: str) -> "DirectRowNorm":
        return cls(ModificationFn(source, "s", allow_reduce=True))


@dataclass(frozen=True)
class OnlineRowNorm:
    """AttentionEngine ``online_func``: prologue / fwd / epilogue over running row scales."""

    rowscales: tuple[str, ...]
    prologue: tuple[tuple[str, ModificationFn], ...]
    fwd: tuple[tuple[str, ModificationFn], ...]
    epilogue: ModificationFn
    direct: DirectRowNorm | None = None


def online(rowscales, prologue: dict[str, str], fwd: dict[str, str], epilogue: str,
           direct: str | None = None) -> OnlineRowNorm:
    return OnlineRowNorm(
        rowscales=tuple(rowscales),
        prologue=tuple((n, ModificationFn(e, None, allow_reduce=True))
                       for n, e in prologue.items()),
        fwd=tuple((n, ModificationFn(e, None, allow_reduce=True)) for n, e in fwd.items()),
        epilogue=ModificationFn(epilogue, "acc", allow_reduce=True),
        direct=DirectRowNorm.from_source(direct) if direct else None,
    )


@dataclass(frozen=True)
class AttentionSpec:
    name: str
    pattern: Pattern
    dims: Dims
    q_mod: ModificationFn | None = None
    k_mod: ModificationFn | None = None
    v_mod: ModificationFn | None = None
    score_mods: tuple[ModificationFn, ...] = ()
    rownorm: OnlineRowNorm | DirectRowNorm | None = None
    output_mod: ModificationFn | None = None
    h_mod: ModificationFn | None = None
    extra_inputs: tuple[ExtraInput, ...] = ()
    kv_shared: bool = False  # MLA extension: V = K[..., :d_v]

    def extras_by_name(self) -> dict[str, ExtraInput]:
        return {e.name: e for e in self.extra_inputs}

    def uses_index_grids(self) -> bool:
        names: set[str] = set()
        for m in self.score_mods:
            names |= m.free_names()
        return bool(names & {"qidx", "kidx"})

    def input_descriptors(self) -> list[ExtraInput]:
        """q, k, v, declared extras and implicit index grids (attention.py:219-233)."""
        out = [ExtraInput("q", ("batch", "heads", "seq_q", "d_qk"), "uniform"),
               ExtraInput("k", ("batch", "heads", "seq_k", "d_qk"), "uniform"),
               ExtraInput("v", ("batch", "heads", "seq_k", "d_v"), "uniform")]
        out += list(self.extra_inputs)
        if self.uses_index_grids():
            out.append(ExtraInput("qidx", (1, 1, "seq_q", 1), "index_q", differentiable=False))
            out.append(ExtraInput("kidx", (1, 1, 1, "seq_k"), "index_k", differentiable=False))
        return out

    def validate(self) -> None:
        """Same rules as attention.py:236-326."""
        seen: set[str] = set()
        for e in self.extra_inputs:
            if e.name in RESERVED_NAMES:
                raise InputError("extra input name is reserved", name=e.name)
            if e.name in seen:
                raise InputError("duplicate extra input", name=e.name)
            seen.add(e.name)
            e.resolve_shape(self.dims)
        consts = set(self.dims.const_env())
        allowed = consts | seen

        def check(fn, input_name, extra_ok=frozenset()):
            if fn is None:
                return
            unknown = fn.free_names() - allowed - {input_name} - set(extra_ok)
            if unknown:
                raise InputError("expression references unknown names",
                                 names=sorted(unknown), source=fn.source)
            if not fn.allow_reduce:
                hooklang.check_elementwise(fn.expr, fn.source)

        check(self.q_mod, "q")
        check(self.k_mod, "k")
        check(self.v_mod, "v")
        check(self.output_mod, "o")
        for m in self.score_mods:
            check(m, "s", extra_ok={"qidx", "kidx"})
        if self.pattern is Pattern.RECURRENT:
            if self.score_mods:
                raise UnsupportedError("recurrent variants do not take score modifications")
            if self.rownorm is not None:
                raise UnsupportedError("recurrent variants fold normalization into h_mod; row "
                                       "normalization is a parallel-pattern feature")
            if self.dims.seq_q != self.dims.seq_k:
                raise InputError("recurrent variants need seq_q == seq_k",
                                 seq_q=self.dims.seq_q, seq_k=self.dims.seq_k)
            check(self.h_mod, "h")
            for e in self.extra_inputs:
                if e.shape[2] != "seq_k":
                    raise InputError("recurrent extras must be per-step tensors on the shared "
                                     "sequence axis", extra=e.name)
        elif self.h_mod is not None:
            raise InputError("h_mod only applies to recurrent variants")
        rn = self.rownorm
        if isinstance(rn, OnlineRowNorm):
            if not rn.rowscales:
                raise InputError("online normalization declares no row scales")
            pro = [n for n, _ in rn.prologue]
            if sorted(pro) != sorted(rn.rowscales):
                raise InputError("prologue must initialize each row scale exactly once",
                                 prologue=pro, rowscales=list(rn.rowscales))
            for n, fn in rn.prologue:
                bad = fn.free_names() - consts
                if bad:
                    raise InputError("prologue reads non-constant names", names=sorted(bad))
            seen_fwd = set(rn.rowscales) | {"s"} | consts
            names = []
            for n, fn in rn.fwd:
                bad = fn.free_names() - seen_fwd
                if bad:
                    raise InputError("fwd reads names not yet defined", assignment=n,
                                     names=sorted(bad))
                seen_fwd.add(n)
                names.append(n)
            for req in ("scores", "rescale"):
                if req not in names:
                    raise InputError(f"fwd must assign {req!r}")
            bad = rn.epilogue.free_names() - ({"acc"} | set(rn.rowscales) | consts)
            if bad:
                raise InputError("epilogue reads names outside acc and final row scales",
                                 names=sorted(bad))
            if rn.direct is not None:
                bad = rn.direct.body.free_names() - ({"s"} | consts)
                if bad:
                    raise InputError("direct form reads unknown names", names=sorted(bad))
        elif isinstance(rn, DirectRowNorm):
            bad = rn.body.free_names() - ({"s"} | consts)
            if bad:
                raise InputError("direct form reads unknown names", names=sorted(bad))
        if self.kv_shared and self.dims.d_v > self.dims.d_qk:
            raise InputError("kv_shared needs d_v <= d_qk", d_qk=self.dims.d_qk,
                             d_v=self.dims.d_v)


def diagonal_scale(h_mod: ModificationFn | None):
    """Per-step scale a_t when h_mod factors as ``h * a_t`` (attention.py:332-369); ``None`` when
    it does not (only stepwise execution applies)."""
    if h_mod is None:
        return hooklang.Num(1.0)
    hname = h_mod.input_name or "h"
    factors: list = []

    def flatten(e):
        if isinstance(e, hooklang.BinOp) and e.op == "*":
            flatten(e.lhs)
            flatten(e.rhs)
        else:
            factors.append(e)

    flatten(h_mod.expr)
    hs = [f for f in factors if isinstance(f, hooklang.Name) and f.name == hname]
    rest = [f for f in factors if not (isinstance(f, hooklang.Name) and f.name == hname)]
    if len(hs) != 1 or any(hname in hooklang.free_names(f) for f in rest):
        return None
    if not rest:
        return hooklang.Num(1.0)
    scale = rest[0]
    for f in rest[1:]:
        scale = hooklang.BinOp("*", scale, f)
    return scale


# ───────────────────────────────── builtins ─────────────────────────────────

def _softmax_rownorm() -> OnlineRowNorm:
    return online(
        rowscales=["m", "l"],
        prologue={"m": "-inf", "l": "0"},
        fwd={"m_new": "max(m, reduceMax(s))",
             "r": "where(m_new == -inf, 1, exp(m - m_new))",
             "p": "where(m_new == -inf, 0, exp(s - m_new))",
             "l": "r * l + reduceSum(p)",
             "m": "m_new",
             "scores": "p",
             "rescale": "r"},
        epilogue="where(l == 0, 0, acc / l)",
        direct="where(reduceMax(s) == -inf, 0, "
               "exp(s - reduceMax(s)) / reduceSum(exp(s - reduceMax(s))))",
    )


def _abssum_rownorm() -> OnlineRowNorm:
    return online(rowscales=["a"], prologue={"a": "0"},
                  fwd={"a": "a + reduceAbssum(s)", "scores": "s", "rescale": "1"},
                  epilogue="acc / clamp(a, 1, inf)",
                  direct="s / clamp(reduceAbssum(s), 1, inf)")


def retention_gammas(heads: int, gamma=None) -> list[float]:
    if gamma is None:
        return [1.0 - 2.0 ** (-5.0 - h) for h in range(heads)]
    if isinstance(gamma, (int, float)):
        return [float(gamma)] * heads
    if len(gamma) != heads:
        raise InputError("gamma list length must equal heads", got=len(gamma), heads=heads)
    return [float(g) for g in gamma]


_SCALE_Q = "q / sqrt(dimqk)"


def _b_softmax(name, dims, **_):
    return AttentionSpec(name, Pattern.PARALLEL, dims, q_mod=mod(_SCALE_Q, "q"),
                         rownorm=_softmax_rownorm())


def _b_sigmoid(name, dims, **_):
    return AttentionSpec(name, Pattern.PARALLEL, dims, q_mod=mod(_SCALE_Q, "q"),
                         score_mods=(mod("sigmoid(s)", "s"),))


def _b_relu(name, dims, **_):
    return AttentionSpec(name, Pattern.PARALLEL, dims, q_mod=mod(_SCALE_Q, "q"),
                         score_mods=(mod("relu(s)", "s"),))


def _b_retention_parallel(name, dims, gamma=None, normalized=True, **_):
    return AttentionSpec(
        name, Pattern.PARALLEL, dims, q_mod=mod(_SCALE_Q, "q"),
        score_mods=(mod("s * mask", "s", ismask=True),),
        rownorm=_abssum_rownorm() if normalized else None,
        extra_inputs=(ExtraInput("mask", (1, "heads", "seq_q", "seq_k"), "causal_decay_mask",
                                 {"gamma": retention_gammas(dims.heads, gamma)},
                                 differentiable=False),))


def _b_retention_recurrent(name, dims, gamma=None, **_):
    return AttentionSpec(
        name, Pattern.RECURRENT, dims, q_mod=mod(_SCALE_Q, "q"), h_mod=mod("h * decay", "h"),
        extra_inputs=(ExtraInput("decay", (1, "heads", "seq_k", 1), "constant_decay",
                                 {"gamma": retention_gammas(dims.heads, gamma)},
                                 differentiable=False),))


def _b_gated_retention(name, dims, **_):
    return AttentionSpec(name, Pattern.RECURRENT, dims, q_mod=mod(_SCALE_Q, "q"),
                         h_mod=mod("h * gate", "h"),
                         extra_inputs=(ExtraInput("gate", ("batch", "heads", "seq_k", 1),
                                                  "unit"),))


def _b_mamba2(name, dims, **_):
    return AttentionSpec(name, Pattern.RECURRENT, dims, k_mod=mod("k * gate", "k"),
                         h_mod=mod("h * decay * gate", "h"),
                         extra_inputs=(ExtraInput("gate", ("batch", "heads", "seq_k", 1), "unit"),
                                       ExtraInput("decay", ("batch", "heads", "seq_k", 1),
                                                  "unit")))


BUILTIN_DIMS: dict[str, tuple[int, int, int]] = {
    "softmax": (32, 128, 128),
    "softmax-deepseek": (16, 192, 128),
    "softmax-diff": (12, 128, 256),
    "sigmoid": (32, 128, 128),
    "relu": (6, 64, 64),
    "retention-parallel": (32, 256, 512),
    "retention-recurrent": (32, 256, 512),
    "gated-retention": (40, 256, 256),
    "mamba2-ssm": (80, 128, 64),
}
_BUILDERS = {
    "softmax": _b_softmax, "softmax-deepseek": _b_softmax, "softmax-diff": _b_softmax,
    "sigmoid": _b_sigmoid, "relu": _b_relu, "retention-parallel": _b_retention_parallel,
    "retention-recurrent": _b_retention_recurrent, "gated-retention": _b_gated_retention,
    "mamba2-ssm": _b_mamba2,
}
BUILTIN_NAMES = tuple(BUILTIN_DIMS)
RECURRENT_BUILTINS = ("retention-recurrent", "gated-retention", "mamba2-ssm")
DEFAULT_SEQ = 2048


def builtin(name: str, *, batch: int = 1, heads: int | None = None, seq_q: int | None = None,
            seq_k: int | None = None, seq: int | None = None, d_qk: int | None = None,
            d_v: int | None = None, scale: float = 1.0, gamma=None, normalized: bool = True,
            heads_kv: int | None = None) -> AttentionSpec:
    """Builtin variant with optional dim overrides (attention.py:707-735)."""
    if name not in _BUILDERS:
        raise UnknownVariantError("not a builtin variant", name=name, known=list(BUILTIN_NAMES))
    h0, dqk0, dv0 = BUILTIN_DIMS[name]
    sq = seq_q if seq_q is not None else (seq if seq is not None else DEFAULT_SEQ)
    sk = seq_k if seq_k is not None else (seq if seq is not None else DEFAULT_SEQ)
    if name in RECURRENT_BUILTINS:
        sk = sq if seq_k is None else sk
    sq = max(1, int(round(sq * scale)))
    sk = max(1, int(round(sk * scale)))
    dims = Dims(batch, heads if heads is not None else h0, sq, sk,
                d_qk if d_qk is not None else dqk0, d_v if d_v is not None else dv0,
                heads_kv=heads_kv)
    spec = _BUILDERS[name](name, dims, gamma=gamma, normalized=normalized)
    spec.validate()
    return spec


def _mentions_exp(fn: ModificationFn | None) -> bool:
    return fn is not None and bool(hooklang.calls(fn.expr) & {"exp", "exp2"})


def causal_mask(spec: AttentionSpec) -> ModificationFn:
    """Additive -inf form when an exponential is downstream, else multiplicative 0/1
    (attention.py:738-774).  Top-left aligned, like the reference."""
    downstream = [spec.output_mod]
    rn = spec.rownorm
    if isinstance(rn, DirectRowNorm):
        downstream.append(rn.body)
    elif isinstance(rn, OnlineRowNorm):
        downstream += [fn for _, fn in rn.fwd] + [rn.epilogue]
        if rn.direct:
            downstream.append(rn.direct.body)
    if any(_mentions_exp(fn) for fn in downstream):
        return mod("where(kidx <= qidx, s, -inf)", "s", ismask=True)
    return mod("s * where(kidx <= qidx, 1, 0)", "s", ismask=True)


def with_causal_mask(spec: AttentionSpec) -> AttentionSpec:
    return replace(spec, score_mods=spec.score_mods + (causal_mask(spec),))


# ───────────────────────────── variant files ─────────────────────────────

_DIM_KEYS = ("batch", "heads", "seq_q", "seq_k", "dqk", "dv")
_MOD_VARS = {"q_mod": "q", "k_mod": "k", "v_mod": "v", "score_mod": "s", "output_mod": "o",
             "h_mod": "h"}
_TOP_KEYS = {"name", "pattern", "dims", "rownorm", "masks", "extras", "notes"} | set(_MOD_VARS)


def _field(doc: dict, key: str, types, where: str, required: bool = True):
    if key not in doc:
        if required:
            raise SchemaError(f"variant file missing field {where}.{key}")
        return None
    v = doc[key]
    if not isinstance(v, types) or isinstance(v, bool):
        raise SchemaError(f"variant field {where}.{key} has wrong type",
                          want=getattr(types, "__name__", str(types)), got=type(v).__name__)
    return v


def _frag(source: str, var, where: str, **kw) -> ModificationFn:
    try:
        return ModificationFn(source, var, **kw)
    except ForgeError as e:
        raise SchemaError(f"variant field {where} does not parse", detail=e.message, **e.context)


def spec_from_dict(doc) -> AttentionSpec:
    """Variant-file JSON → AttentionSpec (variantfile.py:66-127), same field-path errors.
    Optional extension keys: ``dims.heads_kv`` and top-level ``kv_shared``."""
    if not isinstance(doc, dict):
        raise SchemaError("variant file must be a JSON object")
    unknown = sorted(set(doc) - _TOP_KEYS - {"kv_shared"})
    if unknown:
        raise SchemaError("variant file has unknown fields", fields=unknown)
    name = _field(doc, "name", str, "$")
    pat = _field(doc, "pattern", str, "$")
    if pat not in ("parallel", "recurrent"):
        raise SchemaError("variant field $.pattern must be 'parallel' or 'recurrent'", got=pat)
    dd = _field(doc, "dims", dict, "$")
    vals = {k: _field(dd, k, int, "dims") for k in _DIM_KEYS}
    hkv = _field(dd, "heads_kv", int, "dims", required=False)
    dims = Dims(vals["batch"], vals["heads"], vals["seq_q"], vals["seq_k"], vals["dqk"],
                vals["dv"], heads_kv=hkv)
    mods = {}
    for f, var in _MOD_VARS.items():
        src = _field(doc, f, str, "$", required=False)
        mods[f] = None if src is None else _frag(src, var, f)
    score_mods = [mods["score_mod"]] if mods["score_mod"] is not None else []
    for i, entry in enumerate(_field(doc, "masks", list, "$", required=False) or []):
        if not isinstance(entry, dict):
            raise SchemaError(f"variant field masks[{i}] must be an object")
        expr = _field(entry, "expr", str, f"masks[{i}]")
        if entry.get("ismask") is not True:
            raise SchemaError(f"variant field masks[{i}].ismask must be true",
                              got=repr(entry.get("ismask")))
        extra = sorted(set(entry) - {"expr", "ismask"})
        if extra:
            raise SchemaError(f"variant field masks[{i}] has unknown fields", fields=extra)
        score_mods.append(_frag(expr, "s", f"masks[{i}]", ismask=True))
    rownorm = None
    rn = _field(doc, "rownorm", dict, "$", required=False)
    if rn is not None:
        rownorm = _rownorm_from_dict(rn)
    extras = [_extra_from_dict(e, i)
              for i, e in enumerate(_field(doc, "extras", list, "$", required=False) or [])]
    spec = AttentionSpec(name, Pattern(pat), dims, q_mod=mods["q_mod"], k_mod=mods["k_mod"],
                         v_mod=mods["v_mod"], score_mods=tuple(score_mods), rownorm=rownorm,
                         output_mod=mods["output_mod"], h_mod=mods["h_mod"],
                         extra_inputs=tuple(extras), kv_shared=bool(doc.get("kv_shared", False)))
    spec.validate()
    return spec


def _rownorm_from_dict(rn: dict):
    if set(rn) == {"direct"}:
        return DirectRowNorm(_frag(_field(rn, "direct", str, "rownorm"), "s", "rownorm.direct",
                                   allow_reduce=True))
    if set(rn) == {"online"}:
        on = _field(rn, "online", dict, "rownorm")
        rs = _field(on, "rowscales", list, "rownorm.online")
        for r in rs:
            if not isinstance(r, str):
                raise SchemaError("rownorm.online.rowscales entries must be strings",
                                  got=type(r).__name__)
        pro = _field(on, "prologue", dict, "rownorm.online")
        fwd = _field(on, "fwd", dict, "rownorm.online")
        epi = _field(on, "epilogue", str, "rownorm.online")
        for part, obj in (("prologue", pro), ("fwd", fwd)):
            for k, v in obj.items():
                if not isinstance(v, str):
                    raise SchemaError(f"variant field rownorm.online.{part}.{k} must be an "
                                      "expression string", got=type(v).__name__)
        extra = sorted(set(on) - {"rowscales", "prologue", "fwd", "epilogue"})
        if extra:
            raise SchemaError("rownorm.online has unknown fields", fields=extra)
        try:
            return online(list(rs), dict(pro), dict(fwd), epi)
        except ForgeError as e:
            raise SchemaError("rownorm.online does not parse", detail=e.message, **e.context)
    raise SchemaError("variant field $.rownorm must have exactly one of the keys 'direct' or "
                      "'online'", got=sorted(rn))


def _extra_from_dict(entry, i: int) -> ExtraInput:
    where = f"extras[{i}]"
    if not isinstance(entry, dict):
        raise SchemaError(f"variant field {where} must be an object")
    unknown = sorted(set(entry) - {"name", "shape", "fill", "fill_params", "differentiable"})
    if unknown:
        raise SchemaError(f"variant field {where} has unknown fields", fields=unknown)
    name = _field(entry, "name", str, where)
    shape = _field(entry, "shape", list, where)
    if len(shape) != 4:
        raise SchemaError(f"variant field {where}.shape must have 4 entries", got=len(shape))
    for tok in shape:
        if not (tok == 1 or (isinstance(tok, str) and tok in _SHAPE_TOKENS)):
            raise SchemaError(f"variant field {where}.shape has a bad token", token=repr(tok))
    fill = entry.get("fill", "uniform")
    if fill not in FILLS:
        raise SchemaError(f"variant field {where}.fill is unknown", got=fill)
    params = entry.get("fill_params", {})
    if not isinstance(params, dict):
        raise SchemaError(f"variant field {where}.fill_params must be an object")
    diff = entry.get("differentiable", True)
    if not isinstance(diff, bool):
        raise SchemaError(f"variant field {where}.differentiable must be a boolean")
    return ExtraInput(name, tuple(shape), fill, dict(params), diff)


def spec_from_text(text: str, source: str = "<variant>") -> AttentionSpec:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise SchemaError("variant file is not valid JSON", source=source, detail=str(e))
    return spec_from_dict(doc)


def load_variant(path: str) -> AttentionSpec:
    try:
        with open(path, encoding="utf-8") as fh:
            return spec_from_text(fh.read(), source=path)
    except FileNotFoundError:
        raise SchemaError("variant file not found", path=path)


def spec_to_dict(spec: AttentionSpec) -> dict:
    """Inverse of ``spec_from_dict`` (score mods without ``ismask`` become ``score_mod`` — only
    one is representable, matching the file format)."""
    d = spec.dims
    doc: dict = {"name": spec.name, "pattern": spec.pattern.value,
                 "dims": {"batch": d.batch, "heads": d.heads, "seq_q": d.seq_q,
                          "seq_k": d.seq_k, "dqk": d.d_qk, "dv": d.d_v}}
    if d.heads_kv is not None:
        doc["dims"]["heads_kv"] = d.heads_kv
    for f in ("q_mod", "k_mod", "v_mod", "output_mod", "h_mod"):
        fn = getattr(spec, f)
        if fn is not None:
            doc[f] = fn.source
    plain = [m for m in spec.score_mods if not m.ismask]
    masks = [m for m in spec.score_mods if m.ismask]
    if len(plain) > 1 or (plain and spec.score_mods.index(plain[0]) != 0):
        raise InputError("variant files carry one score_mod ahead of the masks")
    if plain:
        doc["score_mod"] = plain[0].source
    if masks:
        doc["masks"] = [{"expr": m.source, "ismask": True} for m in masks]
    rn = spec.rownorm
    if isinstance(rn, DirectRowNorm):
        doc["rownorm"] = {"direct": rn.body.source}
    elif isinstance(rn, OnlineRowNorm):
        doc["rownorm"] = {"online": {
            "rowscales": list(rn.rowscales),
            "prologue": {n: f.source for n, f in rn.prologue},
            "fwd": {n: f.source for n, f in rn.fwd},
            "epilogue": rn.epilogue.source}}
    if spec.extra_inputs:
        doc["extras"] = [{"name": e.name, "shape": list(e.shape), "fill": e.fill,
                          "fill_params": dict(e.fill_params),
                          "differentiable": e.differentiable} for e in spec.extra_inputs]
    if spec.kv_shared:
        doc["kv_shared"] = True
    return doc


def from_reference(ref_spec) -> AttentionSpec:
    """Convert an ``attnforge.attention.AttentionSpec`` (duck-typed) into this API's spec."""
    if isinstance(ref_spec, AttentionSpec):
        return ref_spec

    def conv(fn):
        if fn is None:
            return None
        return ModificationFn(fn.source, fn.input_name, ismask=bool(fn.ismask),
                              allow_reduce=bool(fn.allow_reduce))

    rn = ref_spec.rownorm
    rownorm = None
    if rn is not None and hasattr(rn, "rowscales"):
        rownorm = OnlineRowNorm(
            rowscales=tuple(rn.rowscales),
            prologue=tuple((n, conv(f)) for n, f in rn.prologue),
            fwd=tuple((n, conv(f)) for n, f in rn.fwd),
            epilogue=conv(rn.epilogue),
            direct=DirectRowNorm(conv(rn.direct.body)) if rn.direct is not None else None)
    elif rn is not None:
        rownorm = DirectRowNorm(conv(rn.body))
    d = ref_spec.dims
    dims = Dims(d.batch, d.heads, d.seq_q, d.seq_k, d.d_qk, d.d_v,
                heads_kv=getattr(d, "heads_kv", None))
    extras = tuple(ExtraInput(e.name, tuple(e.shape), e.fill, dict(e.fill_params),
                              bool(e.differentiable)) for e in ref_spec.extra_inputs)
    pattern = Pattern(getattr(ref_spec.pattern, "value", ref_spec.pattern))
    spec = AttentionSpec(ref_spec.name, pattern, dims, conv(ref_spec.q_mod),
                         conv(ref_spec.k_mod), conv(ref_spec.v_mod),
                         tuple(conv(m) for m in ref_spec.score_mods), rownorm,
                         conv(ref_spec.output_mod), conv(ref_spec.h_mod), extras,
                         kv_shared=bool(getattr(ref_spec, "kv_shared", False)))
    spec.validate()
    return spec


def is_softmax_rownorm(rn) -> bool:
    """True when an online rownorm is (structurally) the builtin softmax protocol."""
    if not isinstance(rn, OnlineRowNorm):
        return False
    ref = _softmax_rownorm()
    return (rn.rowscales == ref.rowscales
            and [(n, f.expr) for n, f in rn.prologue] == [(n, f.expr) for n, f in ref.prologue]
            and [(n, f.expr) for n, f in rn.fwd] == [(n, f.expr) for n, f in ref.fwd]
            and rn.epilogue.expr == ref.epilogue.expr)


_ = math  # keep import (used by callers via spec.math in notebooks)
