"""HostPipeline (host buffers, H2D / kernels / D2H overlapped over unit chunks) must return
exactly what the device-resident API returns: every (batch, KV-head) unit is computed by the same
kernels with the same deterministic schedule, so the comparison is bitwise."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import spec as S  # noqa: E402
from paper_2502_15349_b200.pipeline import HostPipeline  # noqa: E402


def _rand(*shape, dtype=torch.bfloat16):
    g = torch.Generator().manual_seed(sum(shape))
    return (torch.rand(*shape, generator=g) * 2 - 1).to(dtype)


@pytest.fixture
def deterministic():
    af.api.use_deterministic_backward(True)
    yield
    af.api.use_deterministic_backward(False)


@pytest.mark.parametrize("b,h,hkv,s", [(3, 8, 2, 512), (1, 8, 4, 384)])
def test_parallel_pipeline_bitwise(b, h, hkv, s, deterministic):
    spec = S.with_causal_mask(S.builtin("softmax", batch=b, heads=h, heads_kv=hkv, seq=s,
                                        d_qk=128, d_v=128))
    host = {"q": _rand(b, h, s, 128).pin_memory(), "k": _rand(b, hkv, s, 128).pin_memory(),
            "v": _rand(b, hkv, s, 128).pin_memory()}
    hdo = _rand(b, h, s, 128).pin_memory()
    out = HostPipeline(spec, max_chunks=4)(host, hdo)
    torch.cuda.synchronize()
    assert len(HostPipeline(spec, max_chunks=4).units) > 1
    dev = {k: v.cuda() for k, v in host.items()}
    o, lse = af.parallel_forward(spec, dev)
    g = af.parallel_backward(spec, dev, o, lse, hdo.cuda())
    assert torch.equal(out["o"], o.cpu())
    assert torch.equal(out["lse"], lse.cpu())
    for n in ("q", "k", "v"):
        assert torch.equal(out[n], g[n].cpu()), n


def test_linear_pipeline_bitwise():
    spec = S.builtin("mamba2-ssm", batch=2, heads=4, seq=512, d_qk=128, d_v=128)
    host = {"q": _rand(2, 4, 512, 128), "k": _rand(2, 4, 512, 128), "v": _rand(2, 4, 512, 128)}
    for e in spec.extra_inputs:
        host[e.name] = 0.5 + 0.45 * _rand(*e.resolve_shape(spec.dims), dtype=torch.float32)
    host = {k: v.pin_memory() for k, v in host.items()}
    hdo = _rand(2, 4, 512, 128).pin_memory()
    out = HostPipeline(spec)(host, hdo)
    torch.cuda.synchronize()
    dev = {k: v.cuda() for k, v in host.items()}
    o = af.linear_forward(spec, dev)
    g = af.linear_backward(spec, dev, hdo.cuda())
    assert torch.equal(out["o"], o.cpu())
    for n in g:
        assert torch.equal(out[n], g[n].cpu()), n


def test_pipeline_rejects_device_inputs():
    spec = S.builtin("softmax", batch=1, heads=1, seq=64, d_qk=64, d_v=64)
    with pytest.raises(af.InputError):
        HostPipeline(spec)({"q": torch.zeros(1, 1, 64, 64, device="cuda")})


def test_mla_pipeline_head_chunks():
    """B = 1 MLA (one latent KV head shared by all heads) chunks over query heads: O, LSE and dQ
    are bitwise the device API's; the latent-KV gradient is the fp32 sum of the per-chunk
    (bf16) partials, so it matches within bf16 rounding of the partials."""
    from paper_2502_15349_b200.configs import mla
    spec = mla(1, 16, 256, 256, causal=True)
    host = {"q": _rand(1, 16, 256, 576).pin_memory(), "k": _rand(1, 1, 256, 576).pin_memory()}
    hdo = _rand(1, 16, 256, 512).pin_memory()
    pipe = HostPipeline(spec, max_chunks=4)
    assert len(pipe.units) == 4
    out = pipe(host, hdo)
    out2 = pipe(host, hdo)  # second call reuses the slot buffers and the accumulator
    torch.cuda.synchronize()
    dev = {k: v.cuda() for k, v in host.items()}
    o, lse = af.parallel_forward(spec, dev)
    g = af.parallel_backward(spec, dev, o, lse, hdo.cuda())
    assert torch.equal(out["o"], o.cpu()) and torch.equal(out["lse"], lse.cpu())
    assert torch.equal(out["q"], g["q"].cpu())
    ref = g["k"].float().cpu()
    err = (out["k"].float() - ref).norm() / ref.norm()
    assert err < 1e-2, err
    assert torch.equal(out2["k"], out["k"])


def test_pipeline_back_to_back_calls(deterministic):
    """Consecutive calls overlap (the next call's copies start under the previous call's last
    kernels, guarded by per-slot events): three calls on different inputs, issued without
    synchronisation, each bitwise equal to the device-resident API."""
    b, h, hkv, s = 2, 4, 2, 384
    spec = S.with_causal_mask(S.builtin("softmax", batch=b, heads=h, heads_kv=hkv, seq=s,
                                        d_qk=128, d_v=128))
    pipe = HostPipeline(spec, max_chunks=4)
    assert len(pipe.units) > 2
    calls = []
    for seed in range(3):
        g = torch.Generator().manual_seed(100 + seed)
        host = {n: (torch.rand(b, hh, s, 128, generator=g) * 2 - 1).bfloat16().pin_memory()
                for n, hh in (("q", h), ("k", hkv), ("v", hkv))}
        hdo = (torch.rand(b, h, s, 128, generator=g) * 2 - 1).bfloat16().pin_memory()
        calls.append((host, hdo))
    outs = [pipe(*c) for c in calls]  # no synchronisation between the calls
    torch.cuda.synchronize()
    for (host, hdo), out in zip(calls, outs):
        dev = {k: v.cuda() for k, v in host.items()}
        o, lse = af.parallel_forward(spec, dev)
        gr = af.parallel_backward(spec, dev, o, lse, hdo.cuda())
        assert torch.equal(out["o"], o.cpu()) and torch.equal(out["lse"], lse.cpu())
        for n in ("q", "k", "v"):
            assert torch.equal(out[n], gr[n].cpu()), n
