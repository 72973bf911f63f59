"""Full-size parity: every BASELINE config runs at its benchmark shape and is checked against the
f64 oracle on slices the oracle finishes in seconds (per (b, h) slice, sampled
query rows for the dense parallel oracle).  Inputs come from ``bench.device_inputs`` — the same
synthetic fills the benchmark times.  Tolerances as in the per-kernel tests: O max-abs 2e-2 and
LSE 1e-3 (parallel / MLA), normwise 2e-2 (linear template, outputs and gradients)."""
import numpy as np
import pytest

from oracle import parallel as OP
from oracle import recurrent as OR

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import configs  # noqa: E402

DEV = torch.device("cuda")


def np64(t):
    return t.double().cpu().numpy()


def nw(got, want):
    got = np.asarray(got, np.float64).reshape(np.shape(want))
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


def test_cfg3_full_size_sampled_rows():
    """B8 H16 S4096 D128 sigmoid + relpos + sliding window 1024: batch elements 0 and 7, all 16
    heads (per-head slopes), rows at the window / diagonal edges."""
    spec = configs.cfg3()
    arrays, _ = bench.device_inputs(spec, DEV, 0)
    o, _ = af.parallel_forward(spec, arrays)
    rows = np.array([0, 1, 1023, 1024, 1025, 2047, 4000, 4095])
    sub = configs.cfg3(batch=1)
    for b in (0, 7):
        a = {"q": np64(arrays["q"][b:b + 1]), "k": np64(arrays["k"][b:b + 1]),
             "v": np64(arrays["v"][b:b + 1])}
        for e in sub.extra_inputs:
            a[e.name] = np64(arrays[e.name])
        want, _ = OP.sampled_forward(sub, a, rows)
        assert np.max(np.abs(np64(o[b, :, rows]) - want[0])) <= 2e-2


def test_cfg4a_full_size_sampled_rows():
    """DeepSeek-V2 MLA prefill B1 H128 S4096 (576/512, causal): sampled rows of four heads."""
    spec = configs.cfg4a()
    arrays, _ = bench.device_inputs(spec, DEV, 0)
    o, lse = af.parallel_forward(spec, arrays)
    rows = np.array([0, 127, 128, 2047, 4095])
    sub = configs.mla(1, 1, 4096, 4096, causal=True)
    k = np64(arrays["k"])
    for h in (0, 41, 100, 127):
        want_o, want_l = OP.sampled_forward(sub, {"q": np64(arrays["q"][:, h:h + 1]), "k": k},
                                            rows)
        assert np.max(np.abs(np64(o[0, h, rows]) - want_o[0, 0])) <= 2e-2
        assert np.max(np.abs(np64(lse[0, h, rows]) - want_l[0, 0])) <= 1e-3


def test_cfg4b_full_size_decode_heads():
    """MLA decode B16 H128 over a 32k latent cache (split-KV + LSE combine): heads of the first
    and last batch elements against the dense oracle over the whole cache."""
    spec = configs.cfg4b()
    arrays, _ = bench.device_inputs(spec, DEV, 0)
    o, lse = af.parallel_forward(spec, arrays)
    sub = configs.mla(1, 1, 1, 32768, causal=False)
    for b in (0, 15):
        k = np64(arrays["k"][b:b + 1])
        for h in (0, 77, 127):
            want_o, want_l = OP.sampled_forward(
                sub, {"q": np64(arrays["q"][b:b + 1, h:h + 1]), "k": k}, np.array([0]))
            assert np.max(np.abs(np64(o[b, h, 0]) - want_o[0, 0, 0])) <= 2e-2
            assert abs(float(lse[b, h, 0]) - float(want_l[0, 0, 0])) <= 1e-3


@pytest.mark.parametrize("key,b,h", [("cfg5a", 3, 0), ("cfg5b", 2, 17)])
def test_linear_full_size_slices(key, b, h):
    """Linear template at S8192 (RetNet 256/256, Mamba2 128/128): forward and VJP of one (b, h)
    slice against the f64 chunked oracle.  RetNet's decay is per head (gamma_h), so its slice is
    head 0 of a one-head spec; Mamba2's gate / decay are per-step inputs, sliced with the head."""
    spec = configs.CONFIGS[key]()
    arrays, dout = bench.device_inputs(spec, DEV, 0)
    o = af.linear_forward(spec, arrays)
    g = af.linear_backward(spec, arrays, dout)
    sub = configs.CONFIGS[key](batch=1, heads=1)

    def cut(t):  # one (b, h) slice; broadcast (size-1) axes stay as they are
        t = t[b:b + 1] if t.shape[0] > 1 else t
        return t[:, h:h + 1] if t.shape[1] > 1 else t
    a = {n: np64(cut(t)) for n, t in arrays.items()}
    want = OR.chunk_forward(sub, a, 64)
    assert nw(np64(o[b:b + 1, h:h + 1]), want) <= 2e-2
    grads = OR.chunk_vjp(sub, a, np64(dout[b:b + 1, h:h + 1]), chunk=64)
    for n in ("q", "k", "v"):
        assert nw(np64(g[n][b:b + 1, h:h + 1]), grads[n]) <= 2e-2, n
