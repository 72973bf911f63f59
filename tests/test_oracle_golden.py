"""Pin the CPU oracle against outputs of the reference implementation itself
(tests/golden/*.npz, produced by tests/golden/make_golden.py from attnforge)."""
import numpy as np
import pytest

import oracle
from oracle import parallel as OP, recurrent as OR
from conftest import golden_cases, load_golden

CASES = golden_cases()


def _close(got, want, tol=1e-9):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape
    scale = max(1.0, float(np.max(np.abs(want)))) if want.size else 1.0
    assert np.array_equal(np.isinf(got), np.isinf(want))
    fin = np.isfinite(want)
    assert np.max(np.abs(got[fin] - want[fin]), initial=0.0) <= tol * scale


def test_fixture_census():
    assert len(CASES) >= 25


@pytest.mark.parametrize("name", CASES)
def test_generate_regenerates_reference_inputs(name):
    spec, arrays, rec = load_golden(name)
    regen = oracle.generate(spec, int(rec["seed"]))
    assert set(regen) == set(arrays)
    for k in arrays:
        assert np.array_equal(regen[k], arrays[k]), k


@pytest.mark.parametrize("name", CASES)
def test_forward_matches_reference(name):
    spec, arrays, rec = load_golden(name)
    if spec.pattern.value == "parallel":
        _close(OP.tiled_forward(spec, arrays, 16, 16), rec["o_tiled"])
        _close(OP.tiled_forward(spec, arrays, 7, 5), rec["o_tiled"])
        _close(OP.naive_forward(spec, arrays), rec["o_naive"])
        if "lse" in rec:
            _close(OP.lse_rows(spec, arrays), rec["lse"])
    else:
        _close(OR.chunk_forward(spec, arrays, 16), rec["o_tiled"], 1e-8)
        _close(OR.step_forward(spec, arrays), rec["o_naive"], 1e-8)


@pytest.mark.parametrize("name", CASES)
def test_vjp_matches_reference_autodiff(name):
    spec, arrays, rec = load_golden(name)
    if "dout" not in rec:
        pytest.skip("no gradient record")
    if spec.pattern.value == "parallel":
        got = OP.parallel_vjp(spec, arrays, rec["dout"])
    else:
        got = OR.chunk_vjp(spec, arrays, rec["dout"], chunk=5)
    for k in [k[2:] for k in rec if k.startswith("g_")]:
        _close(got[k], rec[f"g_{k}"], 1e-8)


def test_streamed_and_keycol_vjps_match_the_dense_vjp():
    """The full-size GPU tests' oracles (row-block streaming; key-column slices given the row
    statistics) reproduce the dense closed-form VJP."""
    import paper_2502_15349_b200 as af
    from paper_2502_15349_b200 import configs
    from oracle import parallel as OP
    for spec in (af.with_causal_mask(af.builtin("softmax", batch=1, heads=4, heads_kv=2, seq=50,
                                                d_qk=16, d_v=16)),
                 configs.cfg3(batch=1, heads=2, seq=40, d=8, window=7),
                 configs.mla(1, 3, 30, 30, True)):
        a = oracle.generate(spec, 1)
        d = spec.dims
        do = np.random.default_rng(0).uniform(-1, 1, (d.batch, d.heads, d.seq_q, d.d_v))
        ref = OP.parallel_vjp(spec, a, do)
        st = OP.streamed_vjp(spec, a, do, block=16)
        assert np.max(np.abs(st["o"] - OP.tiled_forward(spec, a, 8, 8))) <= 1e-12
        for n in ref:
            assert np.max(np.abs(st[n] - ref[n])) <= 1e-12, (spec.name, n)
        if "lse" in st:
            J = np.array([0, 3, 17, 29])
            kc = OP.keycols_softmax_vjp(spec, a, do, st["o"], st["lse"], J)
            for n in kc:
                assert np.max(np.abs(kc[n] - ref[n][:, :, J])) <= 1e-12, (spec.name, n)
