"""Measured tile scheduling on the B200 (schedule.py; the reference's ``schedule --mode measured``
flow, commands.py:200-219 / scheduling.py:256-313): every candidate configuration is timed with
the real kernels, the fastest is recorded, and launches of that spec then use it — with results
that stay within the parity tolerance of the default configuration."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import api, configs, schedule  # noqa: E402


def rnd(*shape, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.rand(*shape, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)


@pytest.mark.parametrize("spec", [configs.cfg2(batch=1, heads=8, heads_kv=2, seq=2048),
                                  configs.cfg4b(batch=4, seq_k=8192),
                                  configs.cfg4a(heads=8, seq=512)],
                         ids=["k1", "mla-decode", "materialised-bwd"])
def test_measured_schedule_picks_and_applies_a_candidate(spec):
    schedule.clear()
    payload = schedule.schedule(spec, mode="measured")
    assert payload["mode"] == "measured" and len(payload["candidates"]) >= 2
    assert all(c["cost"] > 0 for c in payload["candidates"])
    best = min(payload["candidates"], key=lambda c: c["cost"])
    assert payload["cost"] == best["cost"]
    assert schedule.tuning(spec) == payload["plan"]
    d = spec.dims
    arrays = {"q": rnd(d.batch, d.heads, d.seq_q, d.d_qk, seed=1),
              "k": rnd(d.batch, d.kv_heads, d.seq_k, d.d_qk, seed=2)}
    if not spec.kv_shared:
        arrays["v"] = rnd(d.batch, d.kv_heads, d.seq_k, d.d_v, seed=3)
    o_tuned, _ = af.parallel_forward(spec, arrays)
    for cand in schedule.make_scheduling_task(spec).candidates:
        with api.tuned(cand.as_dict()):
            o, _ = af.parallel_forward(spec, arrays)
        err = (o.float() - o_tuned.float()).abs().max().item()
        assert err <= 2e-2, (cand, err)
    schedule.clear()
