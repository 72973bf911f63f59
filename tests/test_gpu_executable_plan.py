"""``integration.B200ExecutablePlan`` in place of the reference's
``lowering.bind_executable(assemble_kernel(spec, tile), plan).run(arrays)`` (lowering.py:971-974):
numpy float64 arrays in, numpy out, on every reference-generated golden fixture (the fixture's
``o_tiled`` is the reference's own output; the tile of the reference plan is irrelevant,
test_engine.py:189-221).  The IR object is duck-typed (``ir.spec``), exactly what attnforge
hands the binder.  Tolerance: the bf16 kernels' O bound, max-abs 2e-2 x max(1, |O|)."""
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import golden_cases, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2502_15349_b200 import integration  # noqa: E402


@pytest.mark.parametrize("name", golden_cases())
def test_bound_b200_plan_reproduces_the_reference_output(name):
    spec, arrays, rec = load_golden(name)
    ir = SimpleNamespace(spec=spec, kind=spec.pattern)
    plan = integration.bind_executable(ir, plan=None)
    got = plan.run(arrays)
    want = rec["o_tiled"]
    assert got.shape == want.shape and got.dtype == np.float64
    scale = max(1.0, float(np.max(np.abs(want))))
    if spec.pattern.value == "parallel":
        assert np.max(np.abs(got - want)) <= 2e-2 * scale, name
    else:  # linear template: normwise (RetNet-like decays make |O| large)
        assert np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30) <= 2e-2, name


def test_numpy_autodiff_grads_match_the_reference_vjp():
    spec, arrays, rec = load_golden("softmax_causal_s96_d32")
    g = integration.autodiff_grads(spec, arrays)
    assert set(g) == {"q", "k", "v"}
    assert all(isinstance(x, np.ndarray) and x.shape == arrays[n].shape for n, x in g.items())
