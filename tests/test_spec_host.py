"""Host-side logic on CPU: hook language, spec validation, builtins, variant files, lowering."""
import math

import numpy as np
import pytest

from oracle import hooks as OH
from paper_2502_15349_b200 import hooklang as H
from paper_2502_15349_b200 import spec as S
from paper_2502_15349_b200 import plan as P
from paper_2502_15349_b200 import errors as E

EXPRS = [
    "exp(s - reduceMax(s)) / reduceSum(exp(s - reduceMax(s)))", "s * where(kidx <= qidx, 1, 0)",
    "q / sqrt(dimqk)", "where(m_new == -inf, 1, exp(m - m_new))", "-x * 2 - -y", "relu(s) * relu(s) / seqk",
    "sigmoid(s - slope * (qidx - kidx) - log(seqk))", "clamp(a, 1, inf)", "30 * tanh(s / 30)",
    "max(m, reduceMax(s))", "min(a, b) + abs(c) - exp2(d)", "1e-3 * x + .5",
]


@pytest.mark.parametrize("src", EXPRS)
def test_parse_print_roundtrip(src):
    node = H.parse(src)
    assert H.parse(H.to_source(node)) == node


@pytest.mark.parametrize("bad", ["1e", "x / 0", "a < b < c", "max(1)", "$", "exp", "(a"])
def test_parse_errors(bad):
    with pytest.raises(E.ParseError):
        H.parse(bad)


@pytest.mark.parametrize("src", [e for e in EXPRS if "reduce" not in e and "where" not in e])
def test_product_fold_matches_oracle_evaluator(src):
    rng = np.random.default_rng(0)
    env = {n: float(rng.uniform(0.2, 2.0)) for n in H.free_names(H.parse(src))}
    env.update({"seqk": 64.0, "dimqk": 16.0})
    got = H.const_value(H.parse(src), env)
    want = float(OH.evaluate(src, dict(env)))
    assert got is not None and math.isclose(got, want, rel_tol=1e-12)


def test_builtin_census_and_dims():
    assert S.BUILTIN_NAMES == ("softmax", "softmax-deepseek", "softmax-diff", "sigmoid", "relu",
                               "retention-parallel", "retention-recurrent", "gated-retention",
                               "mamba2-ssm")
    sp = S.builtin("softmax-deepseek")
    assert (sp.dims.heads, sp.dims.d_qk, sp.dims.d_v, sp.dims.seq_q) == (16, 192, 128, 2048)
    assert S.retention_gammas(2) == [1 - 2 ** -5, 1 - 2 ** -6]


def test_causal_mask_form_follows_downstream_exp():
    assert S.causal_mask(S.builtin("softmax")).source == "where(kidx <= qidx, s, -inf)"
    assert S.causal_mask(S.builtin("sigmoid")).source == "s * where(kidx <= qidx, 1, 0)"


def test_validation_errors():
    with pytest.raises(E.InputError):
        S.AttentionSpec("x", S.Pattern.PARALLEL, S.Dims(1, 1, 4, 4, 2, 2),
                        score_mods=(S.mod("s + zz", "s"),)).validate()
    with pytest.raises(E.UnsupportedError):
        S.AttentionSpec("x", S.Pattern.RECURRENT, S.Dims(1, 1, 4, 4, 2, 2),
                        score_mods=(S.mod("s", "s"),)).validate()
    with pytest.raises(E.InputError):
        S.Dims(1, 0, 4, 4, 2, 2)
    with pytest.raises(E.InputError):
        S.Dims(1, 4, 4, 4, 2, 2, heads_kv=3)


def test_variant_file_errors_name_the_field():
    with pytest.raises(E.SchemaError, match="dims"):
        S.spec_from_dict({"name": "x", "pattern": "parallel", "dims": {"batch": 1}})
    with pytest.raises(E.SchemaError):
        S.spec_from_text("{not json")


def test_spec_roundtrip_through_variant_dict():
    sp = S.with_causal_mask(S.builtin("sigmoid", heads=2, seq=64, d_qk=16, d_v=16))
    assert S.spec_to_dict(S.spec_from_dict(S.spec_to_dict(sp))) == S.spec_to_dict(sp)


def test_lowering_classifies_bench_configs():
    cfg2 = S.with_causal_mask(S.builtin("softmax", batch=8, heads=32, heads_kv=8, seq=8192))
    pl = P.plan_parallel(cfg2)
    assert pl.family == P.FAMILY_SOFTMAX and pl.band.causal == 1 and pl.band.diag_offset == 0
    assert math.isclose(pl.scale, 128 ** -0.5)
    doc = {"name": "cfg3", "pattern": "parallel",
           "dims": {"batch": 8, "heads": 16, "seq_q": 4096, "seq_k": 4096, "dqk": 128, "dv": 128},
           "q_mod": "q / sqrt(dimqk)",
           "score_mod": "sigmoid(s - slope * (qidx - kidx) - log(seqk))",
           "masks": [{"expr": "s * where(kidx <= qidx, 1, 0)", "ismask": True},
                     {"expr": "s * where(qidx - kidx < 1024, 1, 0)", "ismask": True}],
           "extras": [{"name": "slope", "shape": [1, "heads", 1, 1], "fill": "constant_decay",
                       "fill_params": {"gamma": [0.1] * 16}, "differentiable": False}]}
    pl = P.plan_parallel(S.spec_from_dict(doc))
    assert (pl.family, pl.act, pl.band.kernel_window, pl.slope_extra) == \
        (P.FAMILY_ELEMENTWISE, P.ACT_SIGMOID, 1024, "slope")
    assert math.isclose(pl.bias, -math.log(4096))
    lp = P.plan_linear(S.builtin("mamba2-ssm", seq=64))
    assert lp.decay_factors == ("decay", "gate") and lp.k_gate == "gate"


def test_online_softmax_fingerprint_accepts_equivalent_spellings():
    capped = S.spec_from_dict({
        "name": "c", "pattern": "parallel",
        "dims": {"batch": 1, "heads": 1, "seq_q": 8, "seq_k": 8, "dqk": 4, "dv": 4},
        "rownorm": {"online": {"rowscales": ["m", "l"], "prologue": {"m": "log(0)", "l": "0"},
                               "fwd": {"m_new": "max(m, reduceMax(s))",
                                       "r": "where(m_new == log(0), 1, exp(m - m_new))",
                                       "p": "where(m_new == log(0), 0, exp(s - m_new))",
                                       "l_new": "r * l + reduceSum(p)", "m": "m_new",
                                       "l": "l_new", "scores": "p", "rescale": "r"},
                               "epilogue": "where(l == 0, 0, acc / l)"}}})
    assert P.is_online_softmax(capped.rownorm, capped.dims.const_env())
    abssum = S.builtin("retention-parallel", seq=8, d_qk=4, d_v=4).rownorm
    assert not P.is_online_softmax(abssum, {})


def test_band_mask_offsets():
    for src, upper, window in (("where(kidx <= qidx, s, -inf)", 0, None),
                               ("where(kidx < qidx, s, -inf)", -1, None),
                               ("where(kidx <= qidx + 3, s, -inf)", 3, None),
                               ("s * where(qidx - kidx < 5, 1, 0)", None, 5),
                               ("s * where(kidx > qidx - 5, 1, 0)", None, 5)):
        band = P.Band()
        P._mask_kind(S.mod(src, "s", ismask=True), {}, band)
        assert (band.upper, band.window) == (upper, window), src


# ───────────── lowering of the §8(f) hook families (CPU: planner only) ─────────────

def _load(name):
    from conftest import load_golden
    return load_golden(name)[0]


def test_squared_relu_post_scale_folds_into_the_argument():
    spec = _load("variant_squared-relu")
    plan = P.plan_parallel(spec)
    d = spec.dims
    assert plan.family == P.FAMILY_ELEMENTWISE and plan.act == P.ACT_RELU2
    # relu(tau s)^2 / seqk == relu(tau s / sqrt(seqk))^2
    assert math.isclose(plan.scale, d.d_qk ** -0.5 / math.sqrt(d.seq_k), rel_tol=1e-12)
    assert plan.band.upper == 0


def test_capped_softmax_is_softmax_with_a_softcap():
    plan = P.plan_parallel(_load("variant_capped-softmax"))
    assert plan.family == P.FAMILY_SOFTMAX
    assert (plan.cap_a, plan.cap_b) == (30.0, 1.0 / 30.0)


def test_retention_parallel_is_the_abssum_family():
    for name in ("tiny_retention-parallel", "tiny_causal_retention-parallel"):
        spec = _load(name)
        plan = P.plan_parallel(spec)
        assert plan.family == P.FAMILY_ABSSUM and plan.normalize and plan.band.upper == 0
        assert plan.decay_extra == "mask"
        assert plan.decay_gammas == tuple(spec.extra_inputs[0].fill_params["gamma"])
    # unnormalised retention: same family, no row norm
    sp = S.builtin("retention-parallel", heads=2, seq=16, d_qk=8, d_v=8, normalized=False)
    assert not P.plan_parallel(sp).normalize


def test_abssum_fingerprint_rejects_softmax_and_vice_versa():
    c = S.builtin("softmax", heads=1, seq=8, d_qk=4, d_v=4)
    r = S.builtin("retention-parallel", heads=1, seq=8, d_qk=4, d_v=4)
    env = c.dims.const_env()
    assert P.is_online_softmax(c.rownorm, env) and not P.is_online_abssum(c.rownorm, env)
    assert P.is_online_abssum(r.rownorm, env) and not P.is_online_softmax(r.rownorm, env)


def test_feature_maps_recognised():
    spec = _load("variant_silu-retention")
    plan = P.plan_linear(spec)
    assert plan.v_map == P.FM_SILU and plan.q_map == P.FM_NONE
    consts = spec.dims.const_env()
    for src, kind in (("relu(q)", P.FM_RELU), ("sigmoid(q) * q", P.FM_SILU), ("exp(q)", P.FM_EXP),
                      ("tanh(q)", P.FM_TANH), ("q * 0.5", P.FM_NONE)):
        assert P._feature_map(S.mod(src, "q"), "q", consts)[0] == kind
    # any other elementwise mod becomes a compiled hook program (af_hook_eval)
    assert P._feature_map(S.mod("q * q", "q"), "q", consts)[0] == P.FM_HOOK
    from paper_2502_15349_b200 import hookvm
    h = hookvm.compile_hook(S.mod("q * sigmoid(w) + qidx / seqq", "q"), ["q", "w"], consts)
    assert h.operands == ("q", "w") and h.ops[-1] == 11  # ... add
    with pytest.raises(E.UnsupportedError):  # reductions are not elementwise
        hookvm.compile_hook(S.mod("q - reduceMax(q)", "q"), ["q"], consts)
    with pytest.raises(E.UnsupportedError):  # unknown names
        hookvm.compile_hook(S.mod("q * z", "q"), ["q"], consts)


def test_every_reference_fixture_lowers():
    from conftest import golden_cases
    for name in golden_cases():
        spec = _load(name)
        (P.plan_parallel if spec.pattern.value == "parallel" else P.plan_linear)(spec)


def test_emit_is_deterministic_for_every_fixture():
    """Kernel-dialect emission of the chosen B200 plan (lowering.code_generation's shape)."""
    from conftest import golden_cases
    import paper_2502_15349_b200 as af
    for name in golden_cases():
        spec = _load(name)
        text = af.code_generation(spec)
        assert text == af.code_generation(spec)
        assert text.startswith(f'kernel "{spec.name}" template ') and text.rstrip().endswith("}")
    from paper_2502_15349_b200 import configs
    for key, make in configs.CONFIGS.items():
        assert "tmem" in af.code_generation(make())


def test_scheduling_task_candidates_and_analytic_mode():
    """Measured scheduling (schedule.py) exposes the kernels' runtime tile configurations as
    candidates; analytic mode returns the library default without touching a GPU."""
    import paper_2502_15349_b200 as af
    from paper_2502_15349_b200 import configs, schedule
    t = schedule.make_scheduling_task(configs.cfg2(batch=1, heads=4, heads_kv=1, seq=1024))
    assert t.kind == "k1" and [c.kv_stages for c in t.candidates] == [0, 1]
    t = schedule.make_scheduling_task(configs.cfg4b(batch=2, seq_k=4096))
    assert t.kind == "mla-decode" and any(c.splits == 8 for c in t.candidates)
    t = schedule.make_scheduling_task(configs.cfg4a(heads=8, seq=256))
    assert t.kind == "materialised-bwd" and len(t.candidates) > 1
    plan = schedule.tile_config_scheduling(t, mode="analytic")
    assert plan.candidate == schedule.Candidate() and plan.cost > 0
    with pytest.raises(af.UnsupportedError):  # measured mode needs a measure callback
        schedule.tile_config_scheduling(t, mode="measured")
    calls = []
    t.measure = lambda c: (calls.append(c), 1.0 if c.head_groups == 4 else 2.0)[1]
    plan = schedule.tile_config_scheduling(t, mode="measured")
    assert plan.candidate.head_groups == 4 and len(calls) == len(t.candidates)
    assert schedule.tuning(t.spec)["head_groups"] == 4
    schedule.clear()
    assert schedule.tuning(t.spec) == {}
