"""The materialised tier of the parallel template (generic.py: engine.run_naive_parallel on the
GPU) for variants the fused kernels do not lower — checked against the float64 oracle:
retention-parallel at its own head dims (256 / 512, attention.py:682), softmax with an additive
materialised bias extra (the reference's _block_view semantics, engine.py:413-420) and its
gradient, an arbitrary (non-declared-fill) decay mask, a head dim without a fused instantiation,
GQA through the tier.  Tolerances: O normwise 1e-2 / max-abs 2e-2 x max(1, |O|), gradients
normwise 2e-2."""
from dataclasses import replace

import numpy as np
import pytest

import oracle
from oracle import parallel as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import api, spec as S  # noqa: E402


def dev(a):
    return {k: torch.tensor(np.ascontiguousarray(v), device="cuda").to(
        torch.bfloat16 if k in "qkv" else torch.float32) for k, v in a.items()}


def rounded(a):
    out = dict(a)
    for k in "qkv":
        out[k] = torch.tensor(a[k]).to(torch.bfloat16).double().numpy()
    return out


def nw(got, want):
    got = np.asarray(got, np.float64).reshape(np.shape(want))
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


def np64(t):
    return t.double().cpu().numpy()


def check(spec, seed=0, grads=True, fd_extras=()):
    assert api.route_parallel(spec)[0] == "generic"
    a = oracle.generate(spec, seed)
    ra = rounded(a)
    d = dev(a)
    o, stat = af.parallel_forward(spec, d)
    want = OP.tiled_forward(spec, ra, 32, 32)
    assert nw(np64(o), want) <= 1e-2
    assert np.max(np.abs(np64(o) - want)) <= 2e-2 * max(1.0, float(np.max(np.abs(want))))
    if OP._classify(spec) == "softmax":
        lse = OP.lse_rows(spec, ra)
        fin = np.isfinite(lse)
        assert np.max(np.abs(np64(stat)[fin] - lse[fin])) <= 1e-3
    if not grads:
        return
    dout = np.random.default_rng(seed + 1).uniform(-1, 1, want.shape)
    g = af.parallel_backward(spec, d, o, stat, torch.tensor(dout, device="cuda"))
    wv = OP.parallel_vjp(spec, ra, dout)
    for n in wv:
        assert nw(np64(g[n]), wv[n]) <= 2e-2, n
    for name in fd_extras:  # central differences of the oracle forward on a few coordinates
        x = ra[name]
        rng = np.random.default_rng(3)
        for _ in range(4):
            c = tuple(int(rng.integers(0, s_)) for s_ in x.shape)
            lo, hi = dict(ra), dict(ra)
            lo[name], hi[name] = x.copy(), x.copy()
            hi[name][c] += 1e-4
            lo[name][c] -= 1e-4
            fd = (np.sum(dout * OP.naive_forward(spec, hi)) -
                  np.sum(dout * OP.naive_forward(spec, lo))) / 2e-4
            assert abs(float(g[name][c]) - fd) <= 2e-2 * max(1.0, abs(fd)), (name, c)


def test_retention_parallel_at_its_default_head_dims():
    spec = af.builtin("retention-parallel", batch=1, heads=2, seq=96)
    assert (spec.dims.d_qk, spec.dims.d_v) == (256, 512)
    check(spec)


def test_softmax_with_a_materialised_bias_extra_and_its_gradient():
    base = af.with_causal_mask(af.builtin("softmax", batch=2, heads=2, seq=80, d_qk=64, d_v=64))
    bias = S.ExtraInput("bias", (1, "heads", "seq_q", "seq_k"), "uniform")
    spec = replace(base, extra_inputs=(bias,),
                   score_mods=(S.mod("s + bias * 2", "s"),) + tuple(base.score_mods))
    check(spec, fd_extras=("bias",))


def test_arbitrary_decay_mask_values_run_materialised():
    spec = af.with_causal_mask(af.builtin("retention-parallel", heads=2, seq=64, d_qk=64,
                                          d_v=64))
    a = oracle.generate(spec, 1)
    a["mask"] = np.random.default_rng(0).uniform(0, 1, a["mask"].shape)
    ra = rounded(a)
    d = dev(a)
    assert api.route_parallel(spec, d)[0] == "generic"
    o = af.run_tiled_parallel(spec, d)
    assert nw(np64(o), OP.tiled_forward(spec, ra, 16, 16)) <= 1e-2


def test_head_dim_without_a_fused_kernel_and_gqa():
    spec = af.with_causal_mask(af.builtin("softmax", batch=1, heads=4, heads_kv=2, seq=100,
                                          d_qk=320, d_v=96))
    check(spec)


def test_unrecognised_online_rownorm_still_raises():
    base = af.builtin("softmax", heads=2, seq=64, d_qk=64, d_v=64)
    rn = replace(base.rownorm, epilogue=S.ModificationFn("acc / (l + 1)", "acc",
                                                          allow_reduce=True))
    with pytest.raises(af.UnsupportedError):
        af.parallel_forward(replace(base, rownorm=rn), dev(oracle.generate(base, 0)))
