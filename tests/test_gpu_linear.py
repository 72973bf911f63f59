"""Parity of the sm_100a linear template (K4 forward, K5 backward) against the float64 oracle
(oracle pinned to the reference's step/chunk executors and unrolled
autodiff in tests/test_oracle_golden.py).  Tolerance: normwise <= 2e-2 for O and
every gradient, no max-abs bound (RetNet gamma ~ 1 makes |O| large)."""
import numpy as np
import pytest

import oracle
from oracle import recurrent as OR

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import spec as S  # noqa: E402


def to_dev(arrays):
    return {k: torch.tensor(np.ascontiguousarray(v), device="cuda").to(
        torch.bfloat16 if k in ("q", "k", "v") else torch.float32) for k, v in arrays.items()}


def rounded(arrays):
    out = dict(arrays)
    for k in ("q", "k", "v"):
        out[k] = torch.tensor(arrays[k]).to(torch.bfloat16).double().numpy()
    return out


def nw(got, want):
    got = np.asarray(got, np.float64).reshape(np.shape(want))
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


CASES = {
    "retention_d128_s384": ("retention-recurrent", dict(batch=1, heads=2, seq=384, d_qk=128, d_v=128)),
    "retention_d256_ragged": ("retention-recurrent", dict(batch=2, heads=1, seq=300, d_qk=256, d_v=256)),
    "mamba2_d128_s300": ("mamba2-ssm", dict(batch=1, heads=2, seq=300, d_qk=128, d_v=128)),
    "mamba2_dk128_dv256": ("mamba2-ssm", dict(batch=1, heads=1, seq=520, d_qk=128, d_v=256)),
    "gated_retention_d256": ("gated-retention", dict(batch=1, heads=2, seq=256, d_qk=256, d_v=256)),
    "retention_single_chunk_tail": ("retention-recurrent", dict(batch=1, heads=1, seq=77, d_qk=128, d_v=128)),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_linear_forward_matches_oracle(case):
    name, kw = CASES[case]
    spec = S.builtin(name, **kw)
    arrays = oracle.generate(spec, seed=7)
    o = af.linear_forward(spec, to_dev(arrays))
    ref = rounded(arrays)
    assert nw(o.double().cpu().numpy(), OR.chunk_forward(spec, ref, 64)) <= 2e-2
    # chunked == stepwise (the reference's own invariant, test_engine.py:208-221)
    assert nw(o.double().cpu().numpy(), OR.step_forward(spec, ref)) <= 2e-2


@pytest.mark.parametrize("case", sorted(CASES))
def test_linear_backward_matches_oracle(case):
    name, kw = CASES[case]
    spec = S.builtin(name, **kw)
    arrays = oracle.generate(spec, seed=8)
    dev = to_dev(arrays)
    rng = np.random.default_rng(3)
    dout = torch.tensor(rng.uniform(-1, 1, (kw["batch"], kw["heads"], kw["seq"], kw["d_v"])),
                        device="cuda").to(torch.bfloat16)
    grads = af.linear_backward(spec, dev, dout)
    want = OR.chunk_vjp(spec, rounded(arrays), dout.double().cpu().numpy(), chunk=64)
    for k, w in want.items():
        assert nw(grads[k].double().cpu().numpy(), w) <= 2e-2, k


def test_run_chunk_recurrent_signature_and_autograd():
    spec = S.builtin("mamba2-ssm", batch=1, heads=2, seq=256, d_qk=128, d_v=128)
    arrays = to_dev(oracle.generate(spec, 1))
    o1 = af.run_chunk_recurrent(spec, arrays, 64)
    o2 = af.run_step_recurrent(spec, arrays)
    assert torch.equal(o1, o2)
    g = af.autodiff_grads(spec, arrays)
    assert set(g) == {"q", "k", "v", "gate", "decay"}
    assert g["gate"].shape == arrays["gate"].shape


def test_nonfactorable_h_mod_raises():
    base = S.builtin("retention-recurrent", heads=1, seq=128, d_qk=128, d_v=128)
    spec = S.AttentionSpec(base.name, base.pattern, base.dims, q_mod=base.q_mod,
                           h_mod=S.mod("h * h", "h"), extra_inputs=base.extra_inputs)
    with pytest.raises(af.UnsupportedError):
        af.run_chunk_recurrent(spec, to_dev(oracle.generate(base, 0)))


@pytest.mark.parametrize("name,dk,dv", [("retention-recurrent", 128, 128), ("mamba2-ssm", 64, 64),
                                        ("gated-retention", 256, 256)])
def test_prompt_state_then_decode_steps(name, dk, dv):
    """linear_forward(return_state) over a prompt, then linear_step token by token, matches the
    f64 stepwise recurrence (engine.run_step_recurrent) over the whole sequence, and the carried
    state matches the chunked forward's final state over the longer sequence."""
    from dataclasses import replace as dreplace
    b, h, s, extra = 2, 3, 200, 3
    full = S.builtin(name, batch=b, heads=h, seq=s + extra, d_qk=dk, d_v=dv)
    a = oracle.generate(full, 8)
    want = OR.step_forward(full, rounded(a))
    prompt = S.builtin(name, batch=b, heads=h, seq=s, d_qk=dk, d_v=dv)

    def cut(arr, lo, hi):
        return {k: (v[:, :, lo:hi] if v.shape[2] > 1 else v) for k, v in arr.items()}

    o, state = af.linear_forward(prompt, to_dev(cut(a, 0, s)), return_state=True)
    assert state.shape == (b, h, dk, dv) and state.dtype == torch.float32
    assert nw(o.double().cpu().numpy(), want[:, :, :s]) <= 2e-2
    one = dreplace(prompt, dims=dreplace(prompt.dims, seq_q=1, seq_k=1))
    for t in range(s, s + extra):
        ot = af.linear_step(one, to_dev(cut(a, t, t + 1)), state)
        assert nw(ot.double().cpu().numpy(), want[:, :, t:t + 1]) <= 2e-2, t
    _, state_full = af.linear_forward(full, to_dev(a), return_state=True)
    assert nw(state.double().cpu().numpy(), state_full.double().cpu().numpy()) <= 1e-2


def test_broadcast_extra_gradient_is_deterministic_and_summed():
    """A gate broadcast over the batch ([1, H, S, 1]): its gradient sums the per-(b, h) terms in a
    fixed order (no atomics) — two calls agree bitwise and match the oracle's axis sum."""
    from dataclasses import replace as dreplace
    base = S.builtin("gated-retention", batch=3, heads=2, seq=300, d_qk=128, d_v=128)
    spec = dreplace(base, extra_inputs=(dreplace(base.extra_inputs[0],
                                                 shape=(1, "heads", "seq_k", 1),
                                                 differentiable=True),))
    arrays = oracle.generate(spec, seed=4)
    assert arrays["gate"].shape == (1, 2, 300, 1)
    dev = to_dev(arrays)
    dout = torch.rand(3, 2, 300, 128, device="cuda").sub(0.5).to(torch.bfloat16)
    g1 = af.linear_backward(spec, dev, dout)
    g2 = af.linear_backward(spec, dev, dout)
    assert torch.equal(g1["gate"], g2["gate"])
    want = OR.chunk_vjp(spec, rounded(arrays), dout.double().cpu().numpy(), chunk=64)
    assert nw(g1["gate"].double().cpu().numpy(), want["gate"]) <= 2e-2


def test_autograd_engine_returns_extra_gradients():
    """AttentionEngine(mamba2)(q, k, v, gate=, decay=): gate.grad / decay.grad are populated with
    what linear_backward computes."""
    spec = S.builtin("mamba2-ssm", batch=1, heads=2, seq=256, d_qk=128, d_v=128)
    dev = to_dev(oracle.generate(spec, 1))
    leaves = {n: t.clone().requires_grad_() for n, t in dev.items()}
    out = af.AttentionEngine(spec)(leaves["q"], leaves["k"], leaves["v"], gate=leaves["gate"],
                                   decay=leaves["decay"])
    dout = torch.rand_like(out)
    out.backward(dout)
    g = af.linear_backward(spec, dev, dout)
    for n in ("q", "k", "v", "gate", "decay"):
        assert leaves[n].grad is not None, n
        assert torch.equal(leaves[n].grad, g[n].to(leaves[n].dtype)), n


def test_zero_decay_factor_resets_the_state_exactly():
    """A per-step factor of exactly 0 (a state reset) stays finite in the log-space kernels and
    matches the stepwise recurrence; a negative factor is reported as unsupported."""
    spec = S.builtin("mamba2-ssm", batch=1, heads=2, seq=300, d_qk=128, d_v=128)
    arrays = oracle.generate(spec, 2)
    arrays["decay"][:, :, [0, 5, 130, 131, 299]] = 0.0
    o = af.run_chunk_recurrent(spec, to_dev(arrays))
    assert nw(o.double().cpu().numpy(), OR.step_forward(spec, rounded(arrays))) <= 2e-2
    arrays["decay"][:, :, 7] = -0.5
    with pytest.raises(af.UnsupportedError):
        af.run_chunk_recurrent(spec, to_dev(arrays))


def test_zero_key_gate_has_finite_gradient():
    """k_mod = k * gate with gate = 0 on some steps (padding masked through a pure key gate): the
    gate gradient is k . dKm from the raw keys — finite and equal to the oracle's — not
    dk_dot / gate.  A differentiable decay factor that is exactly 0 yields a non-finite gradient
    at that step only (d log a / a); every other gradient stays finite and correct."""
    doc = {"name": "key-gated-retention", "pattern": "recurrent",
           "dims": {"batch": 1, "heads": 2, "seq_q": 300, "seq_k": 300, "dqk": 128, "dv": 128},
           "q_mod": "q / sqrt(dimqk)", "k_mod": "k * gate", "h_mod": "h * decay",
           "extras": [{"name": "gate", "shape": ["batch", "heads", "seq_k", 1], "fill": "unit",
                       "differentiable": True},
                      {"name": "decay", "shape": ["batch", "heads", "seq_k", 1], "fill": "unit",
                       "differentiable": True}]}
    spec = S.spec_from_dict(doc)
    arrays = oracle.generate(spec, seed=6)
    arrays["gate"][:, :, [0, 1, 64, 200, 299]] = 0.0
    dev = to_dev(arrays)
    dout = torch.rand(1, 2, 300, 128, device="cuda").sub(0.5).to(torch.bfloat16)
    g = af.linear_backward(spec, dev, dout)
    assert bool(torch.isfinite(g["gate"]).all())
    want = OR.chunk_vjp(spec, rounded(arrays), dout.double().cpu().numpy(), chunk=64)
    for n in ("gate", "decay", "q", "k", "v"):
        assert nw(g[n].double().cpu().numpy(), want[n]) <= 2e-2, n
    arrays["decay"][:, :, 7] = 0.0
    g = af.linear_backward(spec, to_dev(arrays), dout)
    bad = ~torch.isfinite(g["decay"]).cpu().numpy()[0, :, :, 0]
    assert bad[:, 7].all() and bad.sum() == 2
    for n in ("gate", "q", "k", "v"):  # (the f64 oracle's log-space VJP is NaN here too)
        assert bool(torch.isfinite(g[n]).all()), n
