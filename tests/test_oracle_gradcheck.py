"""Oracle-side finite-difference gradcheck (engine.finite_diff_check restated, engine.py:651-706):
the closed-form VJPs the GPU backward is compared against are themselves checked against central
differences of the float64 forward — every builtin at the reference test's own shape
(test_acceptance.py:174-191), their causal forms, and the cfg3-style variant."""
import pytest

import oracle
from oracle.gradcheck import finite_diff_check
import paper_2502_15349_b200 as af
from paper_2502_15349_b200 import configs
from paper_2502_15349_b200.spec import BUILTIN_DIMS, Pattern

EXPECTED_WRT = {"mamba2-ssm": {"q", "k", "v", "gate", "decay"},
                "gated-retention": {"q", "k", "v", "gate"}}


@pytest.mark.parametrize("name", sorted(BUILTIN_DIMS))
def test_builtin_vjp_matches_central_differences(name):
    spec = af.builtin(name, batch=1, heads=1, seq_q=8, seq_k=8, d_qk=4, d_v=4)
    ok, reports = finite_diff_check(spec, oracle.generate(spec, 5), eps=1e-5, rel_tol=1e-5)
    assert {r.name for r in reports} == EXPECTED_WRT.get(name, {"q", "k", "v"})
    for r in reports:
        assert r.max_rel_err <= 1e-5, (name, r)
    assert ok
    if spec.pattern is Pattern.PARALLEL:
        cspec = af.with_causal_mask(spec)
        ok, reports = finite_diff_check(cspec, oracle.generate(cspec, 6))
        assert ok, (name, reports)


def test_sigmoid_relpos_swa_variant_vjp_and_sampled_mode():
    spec = configs.cfg3(batch=1, heads=2, seq=12, d=4, window=5)
    arrays = oracle.generate(spec, 2)
    ok, reports = finite_diff_check(spec, arrays, sample_per_tensor=20, seed=1)
    assert ok, reports
    assert all(r.checked == 20 for r in reports)


def test_gqa_grads_sum_over_the_group():
    spec = af.with_causal_mask(af.builtin("softmax", batch=1, heads=4, heads_kv=2, seq=6,
                                          d_qk=3, d_v=3))
    ok, reports = finite_diff_check(spec, oracle.generate(spec, 4))
    assert ok, reports
