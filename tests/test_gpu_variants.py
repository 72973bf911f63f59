"""Every reference-generated fixture (tests/golden: all 9 builtins, causal variants, the three
packaged variant files, cfg-style variants) through the bf16 sm_100a kernels.

For each fixture the spec either lowers — then forward (and backward with the fixture's own dO)
must match the float64 oracle evaluated on the bf16-rounded inputs (the oracle itself is pinned to
the fixture by tests/test_oracle_golden.py) — or it raises ``UnsupportedError`` through the public
API (no silent fallback).  Tolerances: O normwise <= 1e-2, max-abs <=
2e-2 * max(1, |O|); LSE max-abs <= 1e-3; gradients normwise <= 2e-2.
"""
import numpy as np
import pytest

from oracle import parallel as OP
from oracle import recurrent as OR
from conftest import golden_cases, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2502_15349_b200 as af  # noqa: E402

DEV = "cuda"


def _dev(arrays: dict) -> dict:
    return {k: torch.tensor(np.ascontiguousarray(v), device=DEV).to(
        torch.bfloat16 if k in ("q", "k", "v") else torch.float32) for k, v in arrays.items()}


def _rounded(arrays: dict) -> dict:
    out = dict(arrays)
    for k in ("q", "k", "v"):
        out[k] = torch.tensor(out[k]).to(torch.bfloat16).double().numpy()
    return out


def _nw(got, want) -> float:
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


def _lowers(spec) -> bool:
    try:
        (af.plan_parallel if spec.pattern.value == "parallel" else af.plan_linear)(spec)
        return True
    except af.UnsupportedError:
        return False


@pytest.mark.parametrize("name", golden_cases())
def test_fixture_through_bf16_kernels(name):
    spec, arrays, rec = load_golden(name)
    dev = _dev({k: v for k, v in arrays.items() if k not in ("qidx", "kidx")})
    parallel = spec.pattern.value == "parallel"
    if not _lowers(spec):
        with pytest.raises(af.UnsupportedError):
            (af.parallel_forward if parallel else af.linear_forward)(spec, dev)
        pytest.skip("variant not lowered (raises UnsupportedError, no fallback)")
    ra = _rounded(arrays)
    dout = rec["dout"] if "dout" in rec else np.random.default_rng(0).uniform(
        -1, 1, size=rec["o_tiled"].shape)
    dout_t = torch.tensor(dout, device=DEV).to(torch.bfloat16)
    dout_r = dout_t.double().cpu().numpy()
    if parallel:
        o, lse = af.parallel_forward(spec, dev)
        want = OP.tiled_forward(spec, ra, 64, 64)
        got = o.double().cpu().numpy()
        assert _nw(got, want) <= 1e-2
        assert np.max(np.abs(got - want)) <= 2e-2 * max(1.0, float(np.max(np.abs(want))))
        if lse is not None and af.plan_parallel(spec).family == 0:  # softmax: the LSE
            wl = OP.lse_rows(spec, ra)
            fin = np.isfinite(wl)
            assert np.max(np.abs(lse.double().cpu().numpy()[fin] - wl[fin]), initial=0.0) <= 1e-3
        elif lse is not None:  # abssum family: the row statistic is sum_j |s_ij|
            z = OP.final_scores(spec, ra)[4]
            wa = np.sum(np.abs(np.where(np.isfinite(z), z, 0.0)), axis=-1)
            assert _nw(lse.double().cpu().numpy(), wa) <= 1e-2
        grads = af.parallel_backward(spec, dev, o, lse, dout_t)
        wg = OP.parallel_vjp(spec, ra, dout_r)
    else:
        o = af.linear_forward(spec, dev)
        want = OR.chunk_forward(spec, ra, 64)
        assert _nw(o.double().cpu().numpy(), want) <= 2e-2
        grads = af.linear_backward(spec, dev, dout_t)
        wg = OR.chunk_vjp(spec, ra, dout_r, chunk=64)
    for n in wg:
        got = grads[n].double().cpu().numpy().reshape(wg[n].shape)
        assert _nw(got, wg[n]) <= 2e-2, n
