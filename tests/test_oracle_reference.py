"""The live reference (attnforge, mounted read-only at /root/reference in the build container)
against this repo's host API and oracle.  Skipped where the reference is absent (the GPU box).

* every builtin (and its causal form) and every packaged variant file converts through
  ``spec.from_reference`` and lowers to a kernel plan (the drop-in boundary accepts the reference's
  own objects);
* the oracle's forwards and VJPs reproduce ``engine.run_tiled_parallel`` /
  ``run_chunk_recurrent`` / ``autodiff_grads`` on the reference's own Philox inputs;
* the oracle's finite-difference check and the reference's ``finite_diff_check``
  (engine.py:651-706) agree.
"""
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC

pytestmark = pytest.mark.skipif(not (REFERENCE_SRC / "attnforge").exists(),
                                reason="reference not mounted")


@pytest.fixture(scope="module")
def ref():
    sys.dont_write_bytecode = True
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    from attnforge import attention as A, engine as E, variantfile as VF
    from importlib import resources
    variants = {}
    vdir = resources.files("attnforge") / "data" / "variants"
    for p in sorted(vdir.iterdir()):
        if p.name.endswith(".json"):
            variants[p.name[:-5]] = VF.spec_from_text(p.read_text(), source=p.name)
    return A, E, variants


def _ref_specs(A, variants):
    out = []
    for name in sorted(A.BUILTIN_NAMES):
        sp = A.builtin(name, batch=1, heads=2, seq_q=24, seq_k=24, d_qk=8, d_v=8)
        out.append((name, sp))
        if sp.pattern is A.Pattern.PARALLEL:
            out.append((name + "+causal", A.with_causal_mask(sp)))
    for name, sp in variants.items():
        out.append(("variant:" + name, sp))
    return out


def test_every_reference_spec_converts_and_lowers(ref):
    A, _, variants = ref
    from paper_2502_15349_b200 import plan as P, spec as S
    for name, rs in _ref_specs(A, variants):
        sp = S.from_reference(rs)
        assert sp.name == rs.name and sp.pattern.value == rs.pattern.value, name
        if sp.pattern is S.Pattern.PARALLEL:
            P.plan_parallel(sp)
        else:
            P.plan_linear(sp)


def test_oracle_matches_live_reference_forward_and_vjp(ref):
    A, E, variants = ref
    import oracle
    from oracle import parallel as OP, recurrent as OR
    from paper_2502_15349_b200 import spec as S
    for name, rs in _ref_specs(A, variants):
        arrays = E.generate(rs, 3).arrays
        sp = S.from_reference(rs)
        mine = oracle.generate(sp, 3)
        for k in arrays:
            assert np.array_equal(arrays[k], mine[k]), (name, k)
        if sp.pattern is S.Pattern.PARALLEL:
            want = E.run_tiled_parallel(rs, arrays, block_q=8, block_k=8)
            got = OP.tiled_forward(sp, arrays, 8, 8)
        else:
            want = E.run_chunk_recurrent(rs, arrays, 8)
            got = OR.chunk_forward(sp, arrays, 8)
        assert np.max(np.abs(got - want)) <= 1e-10, name
        if rs.dims.seq_q > 64:
            continue
        g_ref = E.autodiff_grads(rs, arrays)
        ones = np.ones_like(want)
        g = (OP.parallel_vjp(sp, arrays, ones) if sp.pattern is S.Pattern.PARALLEL
             else OR.chunk_vjp(sp, arrays, ones, chunk=8))
        for n, gr in g_ref.items():
            assert n in g, (name, n)
            err = np.max(np.abs(g[n] - gr)) / max(1.0, np.max(np.abs(gr)))
            assert err <= 1e-8, (name, n, err)


def test_gradcheck_agrees_with_reference_finite_diff_check(ref):
    A, E, _ = ref
    import oracle
    from oracle.gradcheck import finite_diff_check
    from paper_2502_15349_b200 import spec as S
    for name in ("softmax", "relu", "mamba2-ssm", "retention-parallel"):
        rs = A.builtin(name, batch=1, heads=1, seq_q=6, seq_k=6, d_qk=3, d_v=3)
        arrays = E.generate(rs, 5).arrays
        ok_ref, rep_ref = E.finite_diff_check(rs, {k: v.copy() for k, v in arrays.items()})
        ok, rep = finite_diff_check(S.from_reference(rs), oracle.generate(S.from_reference(rs), 5))
        assert ok and ok_ref, name
        assert {r.name for r in rep} == {r.name for r in rep_ref}, name
