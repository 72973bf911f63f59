"""Parity of K3 (MLA: Dqk=576, Dv=512, one latent head, V = K[:, :512]) against the f64 oracle
(the oracle expands the latent head and aliases V to the first 512 columns)."""
from dataclasses import replace

import numpy as np
import pytest

from oracle import parallel as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import spec as S  # noqa: E402


def mla_spec(b, h, sq, sk, causal):
    sp = replace(S.builtin("softmax", batch=b, heads=h, heads_kv=1, seq_q=sq, seq_k=sk, d_qk=576,
                           d_v=512), kv_shared=True)
    return S.with_causal_mask(sp) if causal else sp


def inputs(b, h, sq, sk, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = (torch.rand(b, h, sq, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(b, 1, sk, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
    return q, k


@pytest.mark.parametrize("b,h,sq,sk,causal", [(1, 4, 300, 300, True), (1, 2, 256, 200, False),
                                               (2, 3, 130, 130, True)])
def test_mla_prefill_matches_oracle(b, h, sq, sk, causal):
    q, k = inputs(b, h, sq, sk, 0)
    o, lse = af.parallel_forward(mla_spec(b, h, sq, sk, causal), {"q": q, "k": k})
    rows = np.arange(sq)
    for bb in range(b):
        for hh in range(h):
            a = {"q": q[bb:bb + 1, hh:hh + 1].double().cpu().numpy(),
                 "k": k[bb:bb + 1].double().cpu().numpy()}
            wo, wl = OP.sampled_forward(mla_spec(1, 1, sq, sk, causal), a, rows)
            got = o[bb, hh].double().cpu().numpy()
            assert np.linalg.norm(got - wo[0, 0]) / np.linalg.norm(wo) <= 1e-2
            assert np.max(np.abs(got - wo[0, 0])) <= 2e-2
            assert np.max(np.abs(lse[bb, hh].double().cpu().numpy() - wl[0, 0])) <= 1e-3


# odd tile counts (the CTA pair's last tile pair has one tile), one key, split tails
@pytest.mark.parametrize("b,h,sk", [(2, 128, 5000), (1, 128, 64), (3, 16, 1000), (1, 128, 1),
                                    (2, 128, 97), (4, 64, 4133), (1, 128, 32)])
def test_mla_decode_matches_oracle(b, h, sk):
    q, k = inputs(b, h, 1, sk, 1)
    o, lse = af.parallel_forward(mla_spec(b, h, 1, sk, False), {"q": q, "k": k})
    assert o.shape == (b, h, 1, 512)
    for bb in range(b):
        for hh in (0, h // 2, h - 1):
            a = {"q": q[bb:bb + 1, hh:hh + 1].double().cpu().numpy(),
                 "k": k[bb:bb + 1].double().cpu().numpy()}
            wo, wl = OP.sampled_forward(mla_spec(1, 1, 1, sk, False), a, np.array([0]))
            assert np.max(np.abs(o[bb, hh, 0].double().cpu().numpy() - wo[0, 0, 0])) <= 2e-2
            assert abs(float(lse[bb, hh, 0]) - float(wl[0, 0, 0])) <= 1e-3


def test_mla_decode_entry_point_shapes():
    q, k = inputs(2, 128, 1, 333, 2)
    o, lse = af.api.mla_decode(q[:, :, 0], k[:, 0], 576 ** -0.5)
    assert o.shape == (2, 128, 512) and lse.shape == (2, 128)
    with pytest.raises(af.ShapeError):
        af.api.mla_decode(q[:, :, 0, :64], k[:, 0], 1.0)


def _normwise(got, want):
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


@pytest.mark.parametrize("b,h,sq,sk,causal", [(1, 4, 300, 300, True), (1, 3, 256, 200, False),
                                               (2, 2, 130, 130, True), (1, 5, 512, 512, True)])
def test_mla_backward_matches_oracle(b, h, sq, sk, causal):
    """K3b: dQ and the latent-cache gradient dK + [dV, 0] (summed over heads) against the f64
    closed-form VJP (tolerance: normwise 2e-2)."""
    q, k = inputs(b, h, sq, sk, 3)
    spec = mla_spec(b, h, sq, sk, causal)
    o, lse = af.parallel_forward(spec, {"q": q, "k": k})
    g = torch.Generator(device="cuda").manual_seed(9)
    dout = (torch.rand(b, h, sq, 512, device="cuda", generator=g) * 2 - 1).bfloat16()
    grads = af.parallel_backward(spec, {"q": q, "k": k}, o, lse, dout)
    assert set(grads) == {"q", "k"}
    want = OP.parallel_vjp(spec, {"q": q.double().cpu().numpy(), "k": k.double().cpu().numpy()},
                           dout.double().cpu().numpy())
    assert _normwise(grads["q"].double().cpu().numpy(), want["q"]) <= 2e-2
    assert _normwise(grads["k"].double().cpu().numpy(), want["k"]) <= 2e-2


def test_mla_backward_deterministic():
    q, k = inputs(1, 8, 384, 384, 4)
    spec = mla_spec(1, 8, 384, 384, True)
    o, lse = af.parallel_forward(spec, {"q": q, "k": k})
    dout = torch.ones_like(o)
    a = af.parallel_backward(spec, {"q": q, "k": k}, o, lse, dout)
    b2 = af.parallel_backward(spec, {"q": q, "k": k}, o, lse, dout)
    assert torch.equal(a["q"], b2["q"]) and torch.equal(a["k"], b2["k"])
