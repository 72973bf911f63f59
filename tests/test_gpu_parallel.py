"""Parity of the sm_100a parallel-template kernels (K1 forward, K2 backward, fp32 path) against
the float64 oracle, through the public API → C ABI.  Run on a B200: ``pytest -m gpu``.

Tolerances (stated per BASELINE.md §2; the oracle runs in f64 on the bf16-rounded inputs):
  bf16 O        normwise ≤ 1e-2 and max-abs ≤ 2e-2 · max(1, max|O_ref|)
  LSE (fp32)    max-abs ≤ 1e-3
  bf16 grads    normwise ≤ 2e-2
  fp32 path     max-abs ≤ 1e-5 · max(1, max|O_ref|)   (cfg1)
"""
import math

import numpy as np
import pytest

import oracle
from oracle import parallel as OP
from conftest import golden_cases, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import spec as S  # noqa: E402

DEV = "cuda"


def to_dev(arrays: dict, dtype=torch.bfloat16) -> dict:
    return {k: torch.tensor(np.ascontiguousarray(v), device=DEV).to(
        dtype if k in ("q", "k", "v") else torch.float32) for k, v in arrays.items()}


def rounded(arrays: dict) -> dict:
    """The f64 values the kernel actually sees (q/k/v rounded to bf16)."""
    out = dict(arrays)
    for k in ("q", "k", "v"):
        if k in out:
            out[k] = torch.tensor(out[k]).to(torch.bfloat16).double().numpy()
    return out


def normwise(got, want) -> float:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


def assert_bf16_out(got, want):
    got = got.double().cpu().numpy()
    assert normwise(got, want) <= 1e-2
    assert np.max(np.abs(got - want)) <= 2e-2 * max(1.0, float(np.max(np.abs(want))))


def assert_lse(got, want):
    got = got.double().cpu().numpy()
    assert np.array_equal(np.isneginf(got), np.isneginf(want))
    fin = np.isfinite(want)
    assert np.max(np.abs(got[fin] - want[fin]), initial=0.0) <= 1e-3


def spec_gqa(name, b, h, hkv, sq, sk, d, causal=True, **kw):
    sp = S.builtin(name, batch=b, heads=h, heads_kv=hkv, seq_q=sq, seq_k=sk, d_qk=d, d_v=d, **kw)
    return S.with_causal_mask(sp) if causal else sp


def sigmoid_swa_spec(b, h, s, d, window, hkv=None):
    doc = {"name": "sigmoid-relpos-swa", "pattern": "parallel",
           "dims": {"batch": b, "heads": h, "seq_q": s, "seq_k": s, "dqk": d, "dv": d},
           "q_mod": "q / sqrt(dimqk)",
           "score_mod": "sigmoid(s - slope * (qidx - kidx) - log(seqk))",
           "masks": [{"expr": "s * where(kidx <= qidx, 1, 0)", "ismask": True},
                     {"expr": f"s * where(qidx - kidx < {window}, 1, 0)", "ismask": True}],
           "extras": [{"name": "slope", "shape": [1, "heads", 1, 1], "fill": "constant_decay",
                       "fill_params": {"gamma": [2 ** (-8 * (i + 1) / h) for i in range(h)]},
                       "differentiable": False}]}
    if hkv is not None:
        doc["dims"]["heads_kv"] = hkv
    return S.spec_from_dict(doc)


def strict_causal_spec(b, h, s, d):
    base = S.builtin("softmax", batch=b, heads=h, seq=s, d_qk=d, d_v=d)
    return S.AttentionSpec(base.name, base.pattern, base.dims, q_mod=base.q_mod,
                           rownorm=base.rownorm,
                           score_mods=(S.mod("where(kidx < qidx, s, -inf)", "s", ismask=True),))


BF16_CASES = {
    # cfg1 shape (B1 H4 S512 D64) on the bf16 kernel
    "softmax_causal_cfg1shape": lambda: spec_gqa("softmax", 1, 4, None, 512, 512, 64),
    # cfg2 at reduced sequence: Llama-3 GQA 4:1, D128
    "softmax_causal_gqa_s1024": lambda: spec_gqa("softmax", 1, 8, 2, 1024, 1024, 128),
    "softmax_noncausal_ragged": lambda: spec_gqa("softmax", 2, 2, 1, 200, 333, 128, causal=False),
    "softmax_causal_ragged_d64": lambda: spec_gqa("softmax", 1, 2, 2, 300, 300, 64),
    "softmax_strict_causal_fully_masked_row": lambda: strict_causal_spec(1, 2, 256, 128),
    # cfg3 at reduced size: sigmoid + relative position + causal + sliding window
    "sigmoid_relpos_swa_s1024": lambda: sigmoid_swa_spec(1, 4, 1024, 128, 256),
    "relu_causal_d64": lambda: spec_gqa("relu", 1, 2, None, 384, 384, 64),
    "sigmoid_noncausal_gqa": lambda: spec_gqa("sigmoid", 1, 4, 2, 256, 256, 128, causal=False),
    # builtins at their own head dims beyond K2's TMEM budget (materialised backward)
    "softmax_deepseek_192_128_gqa": lambda: S.with_causal_mask(S.builtin(
        "softmax-deepseek", batch=1, heads=4, heads_kv=2, seq=384, d_qk=192, d_v=128)),
    "softmax_diff_128_256_ragged": lambda: S.with_causal_mask(S.builtin(
        "softmax-diff", batch=2, heads=2, seq=300, d_qk=128, d_v=256)),
    # retention-parallel: causal decay mask synthesised in-kernel + abssum-clamp rows
    "retention_parallel_s512_d128": lambda: S.builtin("retention-parallel", batch=1, heads=4,
                                                      seq=512, d_qk=128, d_v=128),
    "squared_relu_causal_d64": lambda: S.spec_from_dict({
        "name": "squared-relu", "pattern": "parallel",
        "dims": {"batch": 1, "heads": 2, "seq_q": 300, "seq_k": 300, "dqk": 64, "dv": 64},
        "q_mod": "q / sqrt(dimqk)", "score_mod": "relu(s) * relu(s) / seqk",
        "masks": [{"expr": "where(kidx <= qidx, s, 0)", "ismask": True}]}),
}


@pytest.mark.parametrize("case", sorted(BF16_CASES))
def test_bf16_forward_matches_oracle(case):
    spec = BF16_CASES[case]()
    arrays = oracle.generate(spec, seed=11)
    o, lse = af.parallel_forward(spec, to_dev(arrays))
    ref = rounded(arrays)
    want = OP.tiled_forward(spec, ref, 128, 128)
    assert_bf16_out(o, want)
    if lse is not None and af.plan_parallel(spec).family == 0:  # softmax rows: LSE
        assert_lse(lse, OP.lse_rows(spec, ref))


@pytest.fixture
def deterministic():
    """Bitwise comparisons across calls need the split (K2a/K2b) backward: the fused 5-GEMM
    kernel adds dQ partials in L2 arrival order (fp32)."""
    af.api.use_deterministic_backward(True)
    yield
    af.api.use_deterministic_backward(False)


@pytest.fixture(params=["fused", "split"])
def bwd_mode(request):
    af.api.use_deterministic_backward(request.param == "split")
    yield request.param
    af.api.use_deterministic_backward(False)


@pytest.mark.parametrize("case", sorted(BF16_CASES))
def test_bf16_backward_matches_oracle(case, bwd_mode):
    spec = BF16_CASES[case]()
    arrays = oracle.generate(spec, seed=12)
    dev = to_dev(arrays)
    o, lse = af.parallel_forward(spec, dev)
    rng = np.random.default_rng(5)
    dout = rng.uniform(-1, 1, size=tuple(o.shape))
    dout_bf = torch.tensor(dout, device=DEV).to(torch.bfloat16)
    grads = af.parallel_backward(spec, dev, o, lse, dout_bf)
    want = OP.parallel_vjp(spec, rounded(arrays), dout_bf.double().cpu().numpy())
    for k in want:
        assert normwise(grads[k].double().cpu().numpy(), want[k]) <= 2e-2, k


def _fp32_ok(spec) -> bool:
    try:
        af.plan_parallel(spec)
    except af.UnsupportedError:
        return False
    return spec.dims.d_qk == spec.dims.d_v and spec.dims.d_qk in (4, 8, 16, 32, 64, 128)


PAR_GOLDEN = [n for n in golden_cases() if load_golden(n)[0].pattern.value == "parallel"]


@pytest.mark.parametrize("name", PAR_GOLDEN)
def test_fp32_path_matches_reference_golden(name):
    """fp32 exact-FFMA kernel vs the reference's own outputs (golden vectors)."""
    spec, arrays, rec = load_golden(name)
    if not _fp32_ok(spec):
        pytest.skip("variant not lowered on the fp32 path (raises UnsupportedError)")
    o, lse = af.parallel_forward(spec, to_dev(arrays, torch.float32), precision="fp32")
    want = rec["o_tiled"]
    got = o.double().cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-5 * max(1.0, float(np.max(np.abs(want))))
    if "lse" in rec and lse is not None:
        fin = np.isfinite(rec["lse"])
        assert np.max(np.abs(lse.double().cpu().numpy()[fin] - rec["lse"][fin]),
                      initial=0.0) <= 1e-5


def test_cfg1_fp32_full():
    """cfg1: causal softmax B1 H4 S512 D64, fp32, 1e-5 vs f64."""
    spec = spec_gqa("softmax", 1, 4, None, 512, 512, 64)
    arrays = oracle.generate(spec, seed=0)
    o, lse = af.parallel_forward(spec, to_dev(arrays, torch.float32), precision="fp32")
    want = OP.tiled_forward(spec, arrays, 64, 64)
    assert np.max(np.abs(o.double().cpu().numpy() - want)) <= 1e-5
    assert np.max(np.abs(lse.double().cpu().numpy() - OP.lse_rows(spec, arrays))) <= 1e-5


def test_cfg2_full_size_sampled_rows():
    """cfg2 at full size (B8 Hq32 Hkv8 S8192 D128, causal) — kernel output checked on sampled
    (b, h, row) positions against the oracle restricted to those rows."""
    spec = spec_gqa("softmax", 8, 32, 8, 8192, 8192, 128)
    g = torch.Generator(device=DEV).manual_seed(0)
    q = (torch.rand(8, 32, 8192, 128, device=DEV, generator=g) * 2 - 1).to(torch.bfloat16)
    k = (torch.rand(8, 8, 8192, 128, device=DEV, generator=g) * 2 - 1).to(torch.bfloat16)
    v = (torch.rand(8, 8, 8192, 128, device=DEV, generator=g) * 2 - 1).to(torch.bfloat16)
    o, lse = af.parallel_forward(spec, {"q": q, "k": k, "v": v})
    rows = np.array([0, 1, 127, 128, 4095, 4096, 8000, 8191])
    for b, h in ((0, 0), (7, 31), (3, 13)):
        sub = S.with_causal_mask(S.builtin("softmax", batch=1, heads=1, seq=8192, d_qk=128,
                                           d_v=128))
        arrays = {"q": q[b:b + 1, h:h + 1].double().cpu().numpy(),
                  "k": k[b:b + 1, h // 4:h // 4 + 1].double().cpu().numpy(),
                  "v": v[b:b + 1, h // 4:h // 4 + 1].double().cpu().numpy()}
        want_o, want_l = OP.sampled_forward(sub, arrays, rows)
        got = o[b, h, rows].double().cpu().numpy()
        assert np.max(np.abs(got - want_o[0, 0])) <= 2e-2
        assert np.max(np.abs(lse[b, h, rows].double().cpu().numpy() - want_l[0, 0])) <= 1e-3


def test_backward_s4096_gqa_group(bwd_mode):
    """Full-sequence backward at S4096 for one GQA group (4 q heads on 1 KV head)."""
    spec = spec_gqa("softmax", 1, 4, 1, 4096, 4096, 128)
    arrays = oracle.generate(spec, seed=21)
    dev = to_dev(arrays)
    o, lse = af.parallel_forward(spec, dev)
    dout = torch.rand(o.shape, device=DEV).sub(0.5).to(torch.bfloat16)
    grads = af.parallel_backward(spec, dev, o, lse, dout)
    want = OP.parallel_vjp(spec, rounded(arrays), dout.double().cpu().numpy())
    for k in ("q", "k", "v"):
        assert normwise(grads[k].double().cpu().numpy(), want[k]) <= 2e-2, k


def test_autograd_module_matches_backward(deterministic):
    spec = spec_gqa("softmax", 1, 4, 2, 256, 256, 128)
    arrays = oracle.generate(spec, seed=3)
    dev = to_dev(arrays)
    q, k, v = (dev[n].clone().requires_grad_() for n in "qkv")
    eng = af.AttentionEngine(spec)
    out = eng(q, k, v)
    dout = torch.rand_like(out)
    out.backward(dout)
    o, lse = af.parallel_forward(spec, dev)
    g = af.parallel_backward(spec, dev, o, lse, dout)
    for name, t in (("q", q), ("k", k), ("v", v)):
        assert torch.equal(t.grad, g[name])


def test_unlowered_variant_raises_not_falls_back():
    """What neither the fused kernels nor the materialised tier lower raises (no CPU path): an
    online row normalisation that is neither softmax nor abssum-clamp."""
    from dataclasses import replace
    spec = S.with_causal_mask(S.builtin("retention-parallel", heads=2, seq=128, d_qk=64, d_v=64))
    arrays = to_dev(oracle.generate(spec, 0))
    af.run_tiled_parallel(spec, arrays)  # the declared causal decay mask lowers (fused)
    base = S.builtin("softmax", heads=2, seq=128, d_qk=64, d_v=64)
    odd = replace(base, rownorm=replace(base.rownorm, epilogue=S.ModificationFn(
        "acc / (l + 1)", "acc", allow_reduce=True)))
    with pytest.raises(af.UnsupportedError):
        af.parallel_forward(odd, to_dev(oracle.generate(base, 0)))


def test_run_tiled_parallel_accepts_reference_signature():
    spec = spec_gqa("softmax", 1, 2, None, 128, 128, 64)
    arrays = to_dev(oracle.generate(spec, 0))
    o1 = af.run_tiled_parallel(spec, arrays, 64, 64)
    o2 = af.run_tiled_parallel(spec, arrays, 16, 128)
    assert torch.equal(o1, o2)
    assert af.bind(spec).run(arrays).shape == o1.shape


def test_bshd_strided_inputs_match_contiguous(deterministic):
    """[B, S, H, D] activations passed as permuted views (element strides, unit feature stride)
    give the same results as contiguous [B, H, S, D] copies — forward and backward."""
    spec = spec_gqa("softmax", 2, 8, 2, 384, 384, 128)
    arrays = oracle.generate(spec, seed=4)
    dev = to_dev(arrays)
    bshd = {n: dev[n].permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3) for n in "qkv"}
    assert not bshd["q"].is_contiguous()
    o1, l1 = af.parallel_forward(spec, dev)
    o2, l2 = af.parallel_forward(spec, bshd)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    dout = torch.rand_like(o1)
    g1 = af.parallel_backward(spec, dev, o1, l1, dout)
    g2 = af.parallel_backward(spec, bshd, o2, l2, dout)
    for n in "qkv":
        assert torch.equal(g1[n], g2[n]), n


def test_nan_inputs_raise_nan_error():
    """The reference raises on NaN in the final output (engine.py:391-395)."""
    spec = spec_gqa("softmax", 1, 2, None, 128, 128, 64)
    dev = to_dev(oracle.generate(spec, seed=1))
    dev["q"][0, 0, 5, 3] = float("nan")
    with pytest.raises(af.NanError):
        af.run_tiled_parallel(spec, dev)


def test_fused_backward_matches_split_and_repeats():
    """The fused 5-GEMM backward against the split (bitwise-deterministic) pair on the same inputs:
    dK / dV are bitwise reproducible across repeated fused calls (no cross-CTA reduction), dQ to
    fp32 rounding of the reduce-add order; both agree with each other to bf16 rounding."""
    spec = spec_gqa("softmax", 2, 8, 2, 1000, 1000, 128)
    dev = to_dev(oracle.generate(spec, seed=21))
    o, lse = af.parallel_forward(spec, dev)
    dout = torch.rand_like(o) * 2 - 1
    g1 = af.parallel_backward(spec, dev, o, lse, dout)
    g2 = af.parallel_backward(spec, dev, o, lse, dout)
    assert torch.equal(g1["k"], g2["k"]) and torch.equal(g1["v"], g2["v"])
    assert normwise(g1["q"].double().cpu(), g2["q"].double().cpu()) <= 1e-3
    af.api.use_deterministic_backward(True)
    try:
        gs = af.parallel_backward(spec, dev, o, lse, dout)
    finally:
        af.api.use_deterministic_backward(False)
    for n in "qkv":
        assert normwise(g1[n].double().cpu(), gs[n].double().cpu()) <= 5e-3, n
