"""Whole-tensor elementwise hooks on the GPU (af_hook_eval): output_mod on both templates and
q/k/v mods outside af_feature_map's fixed forms, forward and VJP, against the float64 oracle.
Gradients of extras read by these hooks are checked against the oracle's VJP where it has one
and otherwise against central differences of the oracle forward (engine.finite_diff_check's
recipe, engine.py:651-706).  Tolerances: O normwise 1e-2, gradients normwise 2e-2."""
from dataclasses import replace

import numpy as np
import pytest

import oracle
from oracle import parallel as OP, recurrent as OR

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import spec as S  # noqa: E402


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


def fd_grad(fwd, arrays, name, dout, eps=1e-4, n=6, seed=0):
    """Central differences of <dout, fwd(arrays)> on n sampled coordinates of arrays[name]."""
    x = arrays[name]
    rng = np.random.default_rng(seed)
    coords = [tuple(rng.integers(0, s) for s in x.shape) for _ in range(n)]
    out = []
    for c in coords:
        a = {k: v.copy() for k, v in arrays.items()}
        a[name][c] += eps
        lp = float(np.sum(dout * fwd(a)))
        a[name][c] -= 2 * eps
        lm = float(np.sum(dout * fwd(a)))
        out.append((lp - lm) / (2 * eps))
    return coords, np.array(out)


def with_extras(spec, extras, **kw):
    return replace(spec, extra_inputs=tuple(spec.extra_inputs) + tuple(extras), **kw)


def test_parallel_output_mod_forward_and_vjp():
    base = af.with_causal_mask(af.builtin("softmax", batch=2, heads=2, seq=192, d_qk=64,
                                          d_v=64))
    spec = with_extras(base, [S.ExtraInput("g", ("batch", "heads", "seq_q", "d_v"), "unit"),
                              S.ExtraInput("c", (1, "heads", 1, "d_v"), "uniform")],
                       output_mod=S.mod("sigmoid(o * g) + c / seqq", "o"))
    a = oracle.generate(spec, 3)
    ra = rounded(a)
    d = dev(a)
    o, lse = af.parallel_forward(spec, d)
    want = OP.tiled_forward(spec, ra, 64, 64)
    assert nw(np64(o), want) <= 1e-2
    dout = np.random.default_rng(1).uniform(-1, 1, want.shape)
    g = af.parallel_backward(spec, d, o, lse, torch.tensor(dout, device="cuda").to(torch.bfloat16))
    wv = OP.parallel_vjp(spec, ra, dout)
    for n in "qkv":
        assert nw(np64(g[n]), wv[n]) <= 2e-2, n

    def fwd(arr):
        return OP.naive_forward(spec, arr)
    for name in ("g", "c"):
        coords, fd = fd_grad(fwd, ra, name, dout)
        got = np.array([float(g[name][c]) for c in coords])
        assert nw(got, fd) <= 2e-2, name


def test_parallel_qmod_with_an_extra_runs_as_a_hook_program():
    base = af.builtin("sigmoid", batch=1, heads=2, seq=160, d_qk=64, d_v=64)
    spec = with_extras(base, [S.ExtraInput("w", (1, "heads", 1, 1), "uniform")],
                       q_mod=S.mod("q * sigmoid(w) / sqrt(dimqk)", "q"))
    a = oracle.generate(spec, 4)
    ra = rounded(a)
    d = dev(a)
    o, lse = af.parallel_forward(spec, d)
    assert nw(np64(o), OP.tiled_forward(spec, ra, 64, 64)) <= 1e-2
    dout = np.random.default_rng(2).uniform(-1, 1, o.shape)
    g = af.autodiff_grads(spec, d, dout=torch.tensor(dout, device="cuda").to(torch.bfloat16))
    wv = OP.parallel_vjp(spec, ra, dout)
    for n in "qkv":
        assert nw(np64(g[n]), wv[n]) <= 2e-2, n
    coords, fd = fd_grad(lambda arr: OP.naive_forward(spec, arr), ra, "w", dout, n=2)
    assert nw(np.array([float(g["w"][c]) for c in coords]), fd) <= 2e-2


def test_linear_output_mod_and_k_mod_hook():
    base = af.builtin("retention-recurrent", batch=1, heads=2, seq=300, d_qk=128, d_v=128)
    # recurrent extras are per-step tensors (attention.py: validate); k * sigmoid(x) is not the
    # kernels' plain key gate, so it runs as a hook program ahead of the chunked kernel
    spec = with_extras(base, [S.ExtraInput("x", (1, "heads", "seq_k", 1), "uniform"),
                              S.ExtraInput("g", ("batch", "heads", "seq_k", 1), "unit")],
                       k_mod=S.mod("k * sigmoid(x)", "k"), output_mod=S.mod("o * g", "o"))
    a = oracle.generate(spec, 5)
    ra = rounded(a)
    d = dev(a)
    o = af.linear_forward(spec, d)
    want = OR.chunk_forward(spec, ra, 64)
    assert nw(np64(o), want) <= 2e-2
    dout = np.random.default_rng(3).uniform(-1, 1, want.shape)
    g = af.linear_backward(spec, d, torch.tensor(dout, device="cuda").to(torch.bfloat16))
    wv = OR.chunk_vjp(spec, ra, dout, chunk=64)
    for n in ("q", "k", "v", "x"):
        assert nw(np64(g[n]), wv[n]) <= 2e-2, n
    inner = OR.chunk_forward(replace(spec, output_mod=None), ra, 64)
    assert nw(np64(g["g"]), np.sum(dout * inner, -1, keepdims=True)) <= 2e-2


def test_autograd_engine_routes_hook_extra_gradients():
    base = af.with_causal_mask(af.builtin("softmax", batch=1, heads=2, seq=128, d_qk=64,
                                          d_v=64))
    spec = with_extras(base, [S.ExtraInput("g", ("batch", "heads", "seq_q", "d_v"), "unit")],
                       output_mod=S.mod("o * g", "o"))
    d = dev(oracle.generate(spec, 6))
    leaves = {n: t.clone().requires_grad_() for n, t in d.items()}
    out = af.AttentionEngine(spec)(leaves["q"], leaves["k"], leaves["v"], g=leaves["g"])
    out.backward(torch.ones_like(out))
    g = af.autodiff_grads(spec, d)
    for n in ("q", "k", "v", "g"):
        assert torch.allclose(leaves[n].grad.float(), g[n].float(), atol=1e-6), n
