"""Lowering: AttentionSpec → kernel plan (the host half of the template boundary).

The reference assembles a sectioned template per variant (``lowering.assemble_kernel``,
lowering.py:459-468) and interprets it per tile.  Here the same hooks are *classified* into one of
the register-level epilogue families the sm_100a kernels implement, plus launch parameters:

parallel template (``ParallelPlan``)
  * ``q_mod`` / ``k_mod``: a compile-time scalar (``q / sqrt(dimqk)``) folded into the scores;
  * mask hooks (``ismask``): band masks recognised from their comparison
    (``kidx <= qidx`` causal, ``qidx - kidx < W`` sliding window, with offsets) → block skipping in
    the kernel plus per-element masking on edge blocks.  The out-of-band value must be the one the
    family ignores (-inf before softmax, 0 after an elementwise activation);
  * rownorm: the online softmax protocol (recognised numerically, so equivalent spellings such as
    the bundled capped-softmax file's ``log(0)`` form also match) → softmax family with LSE;
    no rownorm → elementwise family ``act(tau*s - slope_h*(qidx-kidx) + bias)`` with
    act ∈ {sigmoid, relu, identity};
  * anything else raises ``UnsupportedError`` — there is no CPU fallback.

recurrent template (``LinearPlan``)
  * ``diagonal_scale(h_mod)`` (attention.py:332-369) must be a product of per-step extras /
    constants; ``k_mod`` may multiply by one per-step extra (Mamba2 ``k * gate``); ``q_mod`` a
    scalar.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import hooklang as H
from .errors import UnsupportedError, InputError
from .spec import (AttentionSpec, DirectRowNorm, OnlineRowNorm, Pattern, diagonal_scale)

FAMILY_SOFTMAX, FAMILY_ELEMENTWISE, FAMILY_ABSSUM = 0, 1, 2
ACT_IDENTITY, ACT_SIGMOID, ACT_RELU, ACT_RELU2 = 0, 1, 2, 3


@dataclass
class Band:
    """Band mask recognised from mask hooks:  keep(i, j) = j <= i + upper  and  i - j < window.

    Kernel parameters (``af_parallel_desc``): causal = upper is set, diag_offset = upper,
    window = window + upper (the kernel's window bound is relative to the diagonal offset)."""

    upper: int | None = None
    window: int | None = None

    def keep(self, i: np.ndarray, j: np.ndarray) -> np.ndarray:
        k = np.ones(np.broadcast_shapes(np.shape(i), np.shape(j)), bool)
        if self.upper is not None:
            k &= j <= i + self.upper
        if self.window is not None:
            k &= (i - j) < self.window
        return k

    @property
    def causal(self) -> int:
        return int(self.upper is not None)

    @property
    def diag_offset(self) -> int:
        return self.upper or 0

    @property
    def kernel_window(self) -> int:
        """The kernels read window <= 0 as "no window": a lower key bound that reaches the
        diagonal offset (e.g. ``where(kidx > qidx, s, -inf)``, keep j > i) is not lowered."""
        if self.window is None:
            return 0
        w = self.window + self.diag_offset
        if w <= 0:
            raise UnsupportedError("mask keeps only keys above the diagonal (lower key bound "
                                   "j > i - window with window + offset <= 0); not lowered",
                                   window=self.window, diag_offset=self.diag_offset)
        return w


FM_NONE, FM_SILU, FM_SIGMOID, FM_RELU, FM_TANH, FM_EXP = range(6)
FM_HOOK = 99  # any other elementwise mod: a compiled hook program (hookvm.py / af_hook_eval)
_FM_BY_FUNC = {"sigmoid": FM_SIGMOID, "relu": FM_RELU, "tanh": FM_TANH, "exp": FM_EXP}


@dataclass
class ParallelPlan:
    spec: AttentionSpec
    family: int
    act: int = ACT_IDENTITY
    scale: float = 1.0
    band: Band = field(default_factory=Band)
    slope_extra: str | None = None  # per-head extra multiplying -(qidx - kidx)
    slope_const: float = 0.0        # constant multiplier of -(qidx - kidx)
    bias: float = 0.0
    q_map: int = FM_NONE            # elementwise feature maps applied ahead of the kernels
    k_map: int = FM_NONE
    v_map: int = FM_NONE
    cap_a: float = 0.0              # softmax family soft-cap s -> cap_a * tanh(cap_b * s)
    cap_b: float = 0.0              # (0 = none; e.g. capped-softmax: 30 * tanh(s / 30))
    # abssum family (retention-parallel): s = tau q.k * gamma_h^(i-j) [j <= i], rows divided by
    # clamp(sum_j |s|, 1, inf) when `normalize`; the decay mask extra is synthesised in-kernel
    decay_extra: str | None = None
    decay_gammas: tuple = ()
    normalize: bool = False
    # compiled whole-tensor hooks: "q"/"k"/"v" for FM_HOOK mods, "o" for output_mod
    hooks: dict = field(default_factory=dict)

    @property
    def has_lse(self) -> bool:
        """Whether the forward emits a per-row statistic: the LSE (softmax family) or the
        row abs-sum a_i (abssum family; the backward's clamp(a_i, 1) and [a_i >= 1])."""
        return self.family in (FAMILY_SOFTMAX, FAMILY_ABSSUM)


@dataclass
class LinearPlan:
    spec: AttentionSpec
    q_scale: float = 1.0
    decay_factors: tuple[str, ...] = ()   # extras whose product (with decay_const) is a_t
    decay_const: float = 1.0
    k_gate: str | None = None             # extra multiplying k (k_mod = k * gate)
    chunk: int = 64
    q_map: int = FM_NONE                  # elementwise feature maps applied ahead of the kernels
    k_map: int = FM_NONE
    v_map: int = FM_NONE
    decay_hint: bool = False              # mild constant decay fills: factorised-decay kernel
    hooks: dict = field(default_factory=dict)  # as ParallelPlan.hooks


# ───────────────────────────── helpers ─────────────────────────────

def _scalar_mod(fn, var: str, consts: dict) -> float:
    """``var * c`` / ``var / c`` / ``c * var`` / bare ``var`` with c a compile-time constant."""
    if fn is None:
        return 1.0
    e = fn.expr
    if isinstance(e, H.Name) and e.name == var:
        return 1.0
    if isinstance(e, H.BinOp) and e.op in "*/":
        for a, b, swap in ((e.lhs, e.rhs, False), (e.rhs, e.lhs, True)):
            if isinstance(a, H.Name) and a.name == var and not (swap and e.op == "/"):
                c = H.const_value(b, consts)
                if c is not None and math.isfinite(c) and c != 0:
                    return c if e.op == "*" else 1.0 / c
    raise UnsupportedError(f"{var}_mod is not a compile-time scalar on this template "
                           "(elementwise feature maps with extras are not lowered yet)",
                           source=fn.source)


def _feature_map(fn, var: str, consts: dict) -> tuple[int, float]:
    """(map kind, scalar) for a q/k/v mod: a compile-time scalar multiple (kind FM_NONE) or one
    of the elementwise maps the feature-map kernel implements, f(var) with f in {var *
    sigmoid(var), sigmoid, relu, tanh, exp}."""
    if fn is None:
        return FM_NONE, 1.0
    try:
        return FM_NONE, _scalar_mod(fn, var, consts)
    except UnsupportedError:
        pass
    e = fn.expr

    def is_var(z):
        return isinstance(z, H.Name) and z.name == var

    if isinstance(e, H.Fn) and e.func in _FM_BY_FUNC and len(e.args) == 1 and is_var(e.args[0]):
        return _FM_BY_FUNC[e.func], 1.0
    if isinstance(e, H.BinOp) and e.op == "*":
        for x, y in ((e.lhs, e.rhs), (e.rhs, e.lhs)):
            if is_var(x) and isinstance(y, H.Fn) and y.func == "sigmoid" and is_var(y.args[0]):
                return FM_SILU, 1.0
    return FM_HOOK, 1.0


def _compile_mods(spec: AttentionSpec, maps: dict, consts: dict) -> dict:
    """Hook programs for the FM_HOOK q/k/v mods and for output_mod (hookvm.compile_hook; the
    inputs a hook may read are its own tensor, the spec's extras and the dims constants)."""
    from . import hookvm
    extras = [e.name for e in spec.extra_inputs]
    hooks = {}
    for var in "qkv":
        if maps.get(f"{var}_map") == FM_HOOK:
            hooks[var] = hookvm.compile_hook(getattr(spec, f"{var}_mod"), [var] + extras, consts)
    if spec.output_mod is not None:
        hooks["o"] = hookvm.compile_hook(spec.output_mod, ["o"] + extras, consts)
    return hooks


def _linear_in_index(e, consts: dict):
    """Return (a, b, c) with e == a*qidx + b*kidx + c for an expression over qidx/kidx/consts,
    or None."""
    if isinstance(e, H.Name):
        if e.name == "qidx":
            return (1.0, 0.0, 0.0)
        if e.name == "kidx":
            return (0.0, 1.0, 0.0)
    c = H.const_value(e, consts)
    if c is not None:
        return (0.0, 0.0, c)
    if isinstance(e, H.Neg):
        r = _linear_in_index(e.operand, consts)
        return None if r is None else tuple(-x for x in r)
    if isinstance(e, H.BinOp):
        l, r = _linear_in_index(e.lhs, consts), _linear_in_index(e.rhs, consts)
        if l is None or r is None:
            return None
        if e.op == "+":
            return tuple(x + y for x, y in zip(l, r))
        if e.op == "-":
            return tuple(x - y for x, y in zip(l, r))
        if e.op == "*":
            if l[0] == l[1] == 0:
                return tuple(l[2] * y for y in r)
            if r[0] == r[1] == 0:
                return tuple(r[2] * x for x in l)
        if e.op == "/" and r[0] == r[1] == 0 and r[2] != 0:
            return tuple(x / r[2] for x in l)
    return None


def _band_from_cond(cond: H.Cmp, consts: dict, band: Band) -> bool:
    """Fold one comparison over qidx/kidx into the band; False when it is not a band bound."""
    l, r = _linear_in_index(cond.lhs, consts), _linear_in_index(cond.rhs, consts)
    if l is None or r is None:
        return False
    a, b, c = (x - y for x, y in zip(l, r))  # a*i + b*j + c  (op)  0
    op = cond.op
    if op in (">", ">="):
        a, b, c = -a, -b, -c
        op = "<" if op == ">" else "<="
    if op not in ("<", "<=") or a != -b or a == 0:
        return False
    # a*(i - j) + c (op) 0 over integer positions.  Strict bounds use ceil(.) - 1 so non-integer
    # constants keep the reference's set (qidx - kidx < 2.5 keeps i - j <= 2).
    if a < 0:  # j - i (op) c/a
        t = c / a
        up = (math.ceil(t - 1e-9) - 1) if op == "<" else math.floor(t + 1e-9)
        band.upper = up if band.upper is None else min(band.upper, up)
    else:      # i - j (op) -c/a  →  keep i - j < w
        t = -c / a
        w = math.ceil(t - 1e-9) if op == "<" else math.floor(t + 1e-9) + 1
        band.window = w if band.window is None else min(band.window, w)
    return True


def _mask_kind(fn, consts: dict, band: Band):
    """Classify a mask hook: returns the out-of-band value (0.0 or -inf) after folding its band
    condition into ``band``; None if unrecognised."""
    e = fn.expr
    if isinstance(e, H.Fn) and e.func == "where" and isinstance(e.args[0], H.Cmp):
        cond, a, b = e.args
        if isinstance(a, H.Name) and a.name == "s":
            out = H.const_value(b, consts)
            if out is not None and (out == 0.0 or out == -math.inf):
                if _band_from_cond(cond, consts, band):
                    return out
    if isinstance(e, H.BinOp) and e.op == "*":
        for x, y in ((e.lhs, e.rhs), (e.rhs, e.lhs)):
            if (isinstance(x, H.Name) and x.name == "s" and isinstance(y, H.Fn)
                    and y.func == "where" and isinstance(y.args[0], H.Cmp)
                    and H.const_value(y.args[1], consts) == 1.0
                    and H.const_value(y.args[2], consts) == 0.0):
                if _band_from_cond(y.args[0], consts, band):
                    return 0.0
    return None


def _run_online(rn: OnlineRowNorm, consts: dict, s: np.ndarray, splits: list[int]) -> np.ndarray:
    """Evaluate an online rownorm protocol on score rows (numpy, for classification only) and
    return the normalised probability rows (acc with V = identity)."""
    rows, n = s.shape
    env0 = dict(consts)
    scales = {name: np.full((rows, 1), float(_np_eval(fn.expr, env0)))
              for name, fn in rn.prologue}
    acc = np.zeros((rows, n))
    start = 0
    for stop in splits + [n]:
        blk = s[:, start:stop]
        env = {**consts, **scales, "s": blk}
        for name, fn in rn.fwd:
            env[name] = _np_eval(fn.expr, env)
        p = np.broadcast_to(np.asarray(env["scores"], float), blk.shape)
        r = np.asarray(env["rescale"], float)
        acc = acc * r
        acc[:, start:stop] += p
        scales = {k: np.asarray(env[k], float) * np.ones((rows, 1)) for k in rn.rowscales}
        start = stop
    out = _np_eval(rn.epilogue.expr, {**consts, **scales, "acc": acc})
    return np.asarray(out, float) * np.ones((rows, n))


def _np_eval(e, env):
    with np.errstate(all="ignore"):
        if isinstance(e, H.Num):
            return e.value
        if isinstance(e, H.Name):
            return env[e.name]
        if isinstance(e, H.Neg):
            return -_np_eval(e.operand, env)
        if isinstance(e, H.BinOp):
            a, b = _np_eval(e.lhs, env), _np_eval(e.rhs, env)
            return {"+": np.add, "-": np.subtract, "*": np.multiply, "/": np.divide}[e.op](
                np.float64(1) * a, b)
        if isinstance(e, H.Cmp):
            a, b = _np_eval(e.lhs, env), _np_eval(e.rhs, env)
            return {"==": np.equal, "!=": np.not_equal, "<": np.less, "<=": np.less_equal,
                    ">": np.greater, ">=": np.greater_equal}[e.op](a, b).astype(float)
        f = e.func
        a = [_np_eval(x, env) for x in e.args]
        one = {"exp": np.exp, "exp2": np.exp2, "log": np.log, "abs": np.abs, "tanh": np.tanh,
               "sigmoid": lambda x: 1 / (1 + np.exp(-np.asarray(x, float))),
               "relu": lambda x: np.maximum(x, 0.0), "sqrt": np.sqrt}
        if f in one:
            return one[f](a[0])
        if f == "reduceSum":
            return np.sum(a[0], axis=-1, keepdims=True)
        if f == "reduceMax":
            return np.max(a[0], axis=-1, keepdims=True)
        if f == "reduceAbssum":
            return np.sum(np.abs(a[0]), axis=-1, keepdims=True)
        if f == "max":
            return np.maximum(a[0], a[1])
        if f == "min":
            return np.minimum(a[0], a[1])
        if f == "clamp":
            return np.clip(a[0], a[1], a[2])
        if f == "where":
            return np.where(np.asarray(a[0]) != 0, a[1], a[2])
    raise InputError("unhandled expression form", form=type(e).__name__)


def is_online_softmax(rn, consts: dict) -> bool:
    """Numerical fingerprint: does this online protocol compute softmax rows for arbitrary
    blockings, including -inf (masked) entries and fully-masked rows (→ 0)?"""
    if not isinstance(rn, OnlineRowNorm):
        return False
    rng = np.random.default_rng(1234)
    s = rng.uniform(-6, 6, size=(6, 24))
    s[1, :9] = -np.inf
    s[2, :] = -np.inf
    s[3, 5:] = -np.inf
    s[4] *= 10.0
    m = np.max(s, axis=-1, keepdims=True)
    with np.errstate(all="ignore"):
        e = np.where(np.isfinite(m), np.exp(s - np.where(np.isfinite(m), m, 0)), 0.0)
        den = e.sum(-1, keepdims=True)
        want = np.where(den == 0, 0.0, e / np.where(den == 0, 1, den))
    try:
        for splits in ([], [1, 2, 9, 17], [12], [3, 6, 9, 12, 15, 18, 21]):
            got = _run_online(rn, consts, s, splits)
            if not np.allclose(got, want, atol=1e-12, rtol=1e-10):
                return False
    except Exception:  # noqa: BLE001 - any evaluation failure means "not softmax"
        return False
    return True


def _strip_act(e, consts: dict):
    """Split ``c * act(inner)`` into (act, inner, fold) where the constant post-scale c is folded
    into the affine inner argument by ``fold`` (relu(x)*c = relu(c x), relu(x)^2*c =
    relu(sqrt(c) x)^2 for c > 0; identity is linear).  Sigmoid admits no post-scale."""
    post = 1.0
    while isinstance(e, H.BinOp) and e.op in "*/":
        cl, cr = H.const_value(e.lhs, consts), H.const_value(e.rhs, consts)
        if cr is not None and cr != 0 and math.isfinite(cr):
            post *= cr if e.op == "*" else 1.0 / cr
            e = e.lhs
        elif cl is not None and e.op == "*" and math.isfinite(cl):
            post *= cl
            e = e.rhs
        else:
            break
    act, inner = ACT_IDENTITY, e
    if isinstance(e, H.Fn) and e.func in ("sigmoid", "relu"):
        act, inner = (ACT_SIGMOID if e.func == "sigmoid" else ACT_RELU), e.args[0]
    elif (isinstance(e, H.BinOp) and e.op == "*" and isinstance(e.lhs, H.Fn)
          and e.lhs.func == "relu" and isinstance(e.rhs, H.Fn) and e.rhs.func == "relu"
          and H.to_source(e.lhs.args[0]) == H.to_source(e.rhs.args[0])):
        act, inner = ACT_RELU2, e.lhs.args[0]
    if post == 1.0:
        return act, inner, 1.0
    if act == ACT_SIGMOID or post <= 0:
        raise UnsupportedError("a constant factor outside sigmoid / a non-positive post-scale is "
                               "not lowered", post=post)
    return act, inner, (math.sqrt(post) if act == ACT_RELU2 else post)


def _affine_score(e, consts: dict, extras: dict):
    """e == tau*s - slope*(qidx - kidx) + bias with slope = const or a per-head extra.
    Returns (tau, slope_const, slope_extra, bias) or None."""
    terms: dict = {}

    def add(key, coef):
        terms[key] = terms.get(key, 0.0) + coef

    def walk(n, sign: float) -> bool:
        if isinstance(n, H.BinOp) and n.op in "+-":
            return walk(n.lhs, sign) and walk(n.rhs, sign if n.op == "+" else -sign)
        if isinstance(n, H.Neg):
            return walk(n.operand, -sign)
        c = H.const_value(n, consts)
        if c is not None:
            add("1", sign * c)
            return True
        if isinstance(n, H.Name) and n.name == "s":
            add("s", sign)
            return True
        lin = _linear_in_index(n, consts)
        if lin is not None and lin[0] == -lin[1]:
            add("d", sign * lin[0])
            add("1", sign * lin[2])
            return True
        if isinstance(n, H.BinOp) and n.op in "*/":
            for x, y in ((n.lhs, n.rhs), (n.rhs, n.lhs)):
                if n.op == "/" and x is n.rhs:
                    continue
                cy = H.const_value(y, consts)
                if isinstance(x, H.Name) and x.name == "s" and cy is not None:
                    add("s", sign * (cy if n.op == "*" else 1.0 / cy))
                    return True
                if isinstance(x, H.Name) and x.name in extras and n.op == "*":
                    lin = _linear_in_index(y, consts)
                    if lin is not None and lin[0] == -lin[1] and lin[2] == 0:
                        add(("x", x.name), sign * lin[0])
                        return True
                    if isinstance(y, H.BinOp) and y.op == "*":
                        pass
            # const * extra * (i - j) forms
            if n.op == "*":
                fs: list = []

                def flat(z):
                    if isinstance(z, H.BinOp) and z.op == "*":
                        flat(z.lhs)
                        flat(z.rhs)
                    else:
                        fs.append(z)

                flat(n)
                coef, ext, lin = 1.0, None, None
                for z in fs:
                    cz = H.const_value(z, consts)
                    if cz is not None:
                        coef *= cz
                    elif isinstance(z, H.Name) and z.name in extras and ext is None:
                        ext = z.name
                    elif lin is None:
                        lin = _linear_in_index(z, consts)
                        if lin is None:
                            return False
                    else:
                        return False
                if lin is not None and lin[0] == -lin[1] and lin[2] == 0:
                    add(("x", ext) if ext else "d", sign * coef * lin[0])
                    return True
        return False

    if not walk(e, 1.0):
        return None
    tau = terms.pop("s", 0.0)
    bias = terms.pop("1", 0.0)
    dcoef = terms.pop("d", 0.0)
    ext = [k for k in terms if isinstance(k, tuple)]
    if terms.keys() - set(ext) or len(ext) > 1 or tau == 0.0:
        return None
    slope_extra, slope_coef = None, 0.0
    if ext:
        slope_extra, slope_coef = ext[0][1], terms[ext[0]]
    # kernel form: z = tau*s - slope*(i - j) + bias  → slope = -coef_of(i - j)
    return tau, -dcoef, slope_extra, -slope_coef, bias


def _plan_parallel(spec: AttentionSpec) -> ParallelPlan:
    plan = _classify_parallel(spec)
    plan.band.kernel_window  # noqa: B018 - raises for a band the kernels cannot express
    return plan


def _classify_parallel(spec: AttentionSpec) -> ParallelPlan:
    if spec.pattern is not Pattern.PARALLEL:
        raise InputError("variant is not a parallel-pattern variant", variant=spec.name)
    spec.validate()
    consts = spec.dims.const_env()
    q_map, q_sc = _feature_map(spec.q_mod, "q", consts)
    k_map, k_sc = _feature_map(spec.k_mod, "k", consts)
    v_map, v_sc = _feature_map(spec.v_mod, "v", consts)
    scale = q_sc * k_sc
    if v_sc != 1.0:  # o is linear in v: a scalar v_mod becomes a one-op hook program
        v_map = FM_HOOK
    maps = dict(q_map=q_map, k_map=k_map, v_map=v_map)
    maps["hooks"] = _compile_mods(spec, maps, consts)
    band = Band()
    plain, mask_vals = [], []
    seen_mask = False
    rn = spec.rownorm
    masks = [m for m in spec.score_mods if m.ismask]
    decay_mods = [m for m in masks if _decay_mask(spec, [m]) is not None]
    if (len(decay_mods) == 1 and len(masks) == len(spec.score_mods)
            and (rn is None or is_online_abssum(rn, consts))):
        # retention-parallel: a causal decay-mask extra (synthesised in-kernel; its zeros above the
        # diagonal make the band causal), further 0/1 band masks, abssum-clamp rows
        dname, gammas = _decay_mask(spec, decay_mods)
        dband = Band(upper=0)
        for m in masks:
            if m is decay_mods[0]:
                continue
            if _mask_kind(m, consts, dband) != 0.0:
                raise UnsupportedError("masks next to a decay mask must zero the score (s*0/1)",
                                       source=m.source)
        return ParallelPlan(spec, FAMILY_ABSSUM, scale=scale, band=dband, decay_extra=dname,
                            decay_gammas=gammas, normalize=rn is not None, **maps)
    for m in spec.score_mods:
        if m.ismask:
            seen_mask = True
            v = _mask_kind(m, consts, band)
            if v is None:
                raise UnsupportedError("mask_mod is not a recognised band mask", source=m.source)
            mask_vals.append(v)
        else:
            if seen_mask:
                raise UnsupportedError("score_mod after a mask_mod is not lowered", source=m.source)
            plain.append(m)
    if rn is not None and is_online_softmax(rn if isinstance(rn, OnlineRowNorm) else None, consts):
        cap = (0.0, 0.0)
        if plain:
            cap = _softcap(plain, consts)
            if cap is None:
                raise UnsupportedError("score_mod ahead of the online softmax must be a soft-cap "
                                       "A * tanh(s * B)", source=plain[0].source)
        if any(v != -math.inf for v in mask_vals):
            raise UnsupportedError("softmax masks must use the additive -inf form")
        return ParallelPlan(spec, FAMILY_SOFTMAX, scale=scale, band=band, cap_a=cap[0],
                            cap_b=cap[1], **maps)
    if isinstance(rn, DirectRowNorm) and _direct_is_softmax(rn, consts):
        if plain or any(v != -math.inf for v in mask_vals):
            raise UnsupportedError("direct softmax with score mods is not lowered")
        return ParallelPlan(spec, FAMILY_SOFTMAX, scale=scale, band=band, **maps)
    if rn is not None:
        raise UnsupportedError("row normalisation is neither online softmax nor absent; the "
                               "abssum-clamp / generic online forms are not lowered yet",
                               variant=spec.name)
    # elementwise family: compose the plain score mods into one expression of s
    expr = H.Name("s")
    for m in plain:
        expr = _substitute(m.expr, "s", expr)
    act, inner, fold = _strip_act(expr, consts)
    extras = {e.name: e for e in spec.extra_inputs}
    aff = _affine_score(inner, consts, extras)
    if aff is None:
        raise UnsupportedError("score_mod is not c*act(a*s + slope*(qidx-kidx) + b)",
                               expr=H.to_source(expr))
    tau, slope_c, slope_x, slope_xc, bias = aff
    if fold != 1.0:
        if slope_x is not None:
            raise UnsupportedError("post-scaled activations with a per-head slope extra are "
                                   "not lowered")
        tau, slope_c, bias = tau * fold, slope_c * fold, bias * fold
    if any(v != 0.0 for v in mask_vals):
        raise UnsupportedError("masks ahead of a norm-free score must zero the score (s*0/1)")
    if slope_x is not None:
        ex = extras[slope_x]
        if tuple(ex.shape) not in ((1, "heads", 1, 1), (1, 1, 1, 1)):
            raise UnsupportedError("relative-position slope extra must be per-head [1,heads,1,1]",
                                   extra=slope_x)
        if slope_c != 0.0:
            raise UnsupportedError("mixed constant and per-head slopes are not lowered")
    if slope_x is not None and slope_xc != 1.0:
        raise UnsupportedError("slope extra must enter with coefficient 1", coef=slope_xc)
    return ParallelPlan(spec, FAMILY_ELEMENTWISE, act=act, scale=scale * tau, band=band,
                        slope_extra=slope_x, slope_const=slope_c, bias=bias, **maps)


def _softcap(mods, consts: dict) -> tuple[float, float] | None:
    """A single score mod of the form ``A * tanh(s * B)`` (or ``tanh(s / C) * A``, constants) —
    the logit soft-cap ahead of the softmax."""
    if len(mods) != 1:
        return None
    e = mods[0].expr
    a = 1.0
    if isinstance(e, H.BinOp) and e.op == "*":
        for x, y in ((e.lhs, e.rhs), (e.rhs, e.lhs)):
            c = H.const_value(x, consts)
            if c is not None and isinstance(y, H.Fn) and y.func == "tanh":
                a, e = c, y
                break
    if not (isinstance(e, H.Fn) and e.func == "tanh"):
        return None
    inner = e.args[0]
    try:
        b = _scalar_mod(type("M", (), {"expr": inner, "source": H.to_source(inner)})(), "s",
                        consts)
    except UnsupportedError:
        return None
    if not (math.isfinite(a) and math.isfinite(b)) or a == 0.0:
        return None
    return a, b


def is_online_abssum(rn, consts: dict) -> bool:
    """Numerical fingerprint of the abssum-clamp rownorm (attention.py:575-586): rows divided by
    clamp(sum |s|, 1, inf), for arbitrary blockings."""
    if not isinstance(rn, OnlineRowNorm):
        return False
    rng = np.random.default_rng(99)
    s = rng.uniform(-0.2, 0.2, size=(5, 24))
    s[1] *= 0.01   # |row| sum < 1: the clamp floor
    s[2, 10:] = 0.0
    s[3] *= 10.0
    a = np.sum(np.abs(s), -1, keepdims=True)
    want = s / np.clip(a, 1.0, None)
    try:
        for splits in ([], [1, 2, 9, 17], [12]):
            if not np.allclose(_run_online(rn, consts, s, splits), want, atol=1e-12, rtol=1e-10):
                return False
    except Exception:  # noqa: BLE001 - any evaluation failure means "not abssum"
        return False
    return True


def _decay_mask(spec: AttentionSpec, mods) -> tuple[str, tuple] | None:
    """A single multiplicative mask ``s * X`` where X is a [1, heads, seq_q, seq_k] extra with the
    reference's causal_decay_mask fill (gamma_h^(i-j) on j <= i, 0 above the diagonal)."""
    if len(mods) != 1:
        return None
    e = mods[0].expr
    extras = {x.name: x for x in spec.extra_inputs}
    if not (isinstance(e, H.BinOp) and e.op == "*"):
        return None
    for x, y in ((e.lhs, e.rhs), (e.rhs, e.lhs)):
        if isinstance(x, H.Name) and x.name == "s" and isinstance(y, H.Name) and y.name in extras:
            ex = extras[y.name]
            if ex.fill == "causal_decay_mask" and tuple(ex.shape) == (1, "heads", "seq_q", "seq_k"):
                g = tuple(float(v) for v in ex.fill_params["gamma"])
                if len(g) == spec.dims.heads and all(0.0 < v <= 1.0 for v in g):
                    return ex.name, g
    return None


def _direct_is_softmax(rn: DirectRowNorm, consts) -> bool:
    rng = np.random.default_rng(7)
    s = rng.uniform(-5, 5, size=(4, 16))
    s[1, :4] = -np.inf
    s[2] = -np.inf
    try:
        got = np.asarray(_np_eval(rn.body.expr, {**consts, "s": s}), float)
    except Exception:  # noqa: BLE001
        return False
    m = np.max(s, -1, keepdims=True)
    with np.errstate(all="ignore"):
        e = np.where(np.isfinite(m), np.exp(s - np.where(np.isfinite(m), m, 0)), 0)
        den = e.sum(-1, keepdims=True)
        want = np.where(den == 0, 0, e / np.where(den == 0, 1, den))
    return bool(np.allclose(got, want, atol=1e-12))


def _substitute(e, name: str, by):
    if isinstance(e, H.Name):
        return by if e.name == name else e
    if isinstance(e, H.Num):
        return e
    if isinstance(e, H.Neg):
        return H.Neg(_substitute(e.operand, name, by))
    if isinstance(e, (H.BinOp, H.Cmp)):
        return type(e)(e.op, _substitute(e.lhs, name, by), _substitute(e.rhs, name, by))
    return H.Fn(e.func, tuple(_substitute(a, name, by) for a in e.args))


def _plan_linear(spec: AttentionSpec, chunk: int = 64) -> LinearPlan:
    if spec.pattern is not Pattern.RECURRENT:
        raise InputError("variant is not a recurrent-pattern variant", variant=spec.name)
    spec.validate()
    consts = spec.dims.const_env()
    scale = diagonal_scale(spec.h_mod)
    if scale is None:
        raise UnsupportedError("h_mod does not factor as h times a per-step scale; only stepwise "
                               "execution applies", h_mod=spec.h_mod.source)
    extras = spec.extras_by_name()
    factors: list = []

    def flat(z):
        if isinstance(z, H.BinOp) and z.op == "*":
            flat(z.lhs)
            flat(z.rhs)
        else:
            factors.append(z)

    flat(scale)
    const, names = 1.0, []
    for f in factors:
        c = H.const_value(f, consts)
        if c is not None:
            const *= c
        elif isinstance(f, H.Name) and f.name in extras:
            names.append(f.name)
        else:
            raise UnsupportedError("per-step scale is not a product of extras and constants",
                                   factor=H.to_source(f))
    k_gate = None
    k_map, k_sc = FM_NONE, 1.0
    if spec.k_mod is not None:
        e = spec.k_mod.expr
        if isinstance(e, H.BinOp) and e.op == "*":
            for x, y in ((e.lhs, e.rhs), (e.rhs, e.lhs)):
                if isinstance(x, H.Name) and x.name == "k" and isinstance(y, H.Name) \
                        and y.name in extras and tuple(extras[y.name].shape)[2:] == ("seq_k", 1):
                    k_gate = y.name  # a per-step key gate: applied inside the kernels
        if k_gate is None:
            k_map, k_sc = _feature_map(spec.k_mod, "k", consts)
    v_map, v_scale = _feature_map(spec.v_mod, "v", consts)
    q_map, q_scale = _feature_map(spec.q_mod, "q", consts)
    maps = dict(q_map=q_map, k_map=k_map, v_map=v_map)
    hooks = _compile_mods(spec, maps, consts)
    hint = 0.5 <= const and all(
        extras[nm].fill == "constant_decay"
        and all(0.5 <= float(g) <= 1.0 for g in extras[nm].fill_params.get("gamma", [0.0]))
        for nm in names)
    # o is linear in q, k and v: scalar mods fold into the output scale
    return LinearPlan(spec, q_scale=q_scale * v_scale * k_sc, decay_factors=tuple(names),
                      decay_const=const, k_gate=k_gate, chunk=chunk, q_map=q_map, k_map=k_map,
                      v_map=v_map, decay_hint=hint, hooks=hooks)


# ───────────────────────────── plan cache ─────────────────────────────
# Lowering classifies hooks numerically (milliseconds of host work); a spec's plan is a pure
# function of the spec, so plans are memoised by the spec's repr (specs may hold unhashable
# fill-parameter dicts).  Bounded, insertion-ordered eviction.
_CACHE: dict = {}
_CACHE_MAX = 256


def _cached(key, make):
    hit = _CACHE.get(key)
    if hit is None:
        hit = make()
        if len(_CACHE) >= _CACHE_MAX:
            _CACHE.pop(next(iter(_CACHE)))
        _CACHE[key] = hit
    return hit


def plan_parallel(spec: AttentionSpec) -> ParallelPlan:
    """Lower a parallel-pattern spec to its kernel plan (memoised; see ``_plan_parallel``)."""
    return _cached(("parallel", repr(spec)), lambda: _plan_parallel(spec))


def plan_linear(spec: AttentionSpec, chunk: int = 64) -> LinearPlan:
    """Lower a recurrent-pattern spec to its kernel plan (memoised; see ``_plan_linear``)."""
    return _cached(("linear", chunk, repr(spec)), lambda: _plan_linear(spec, chunk))
