"""Reference-side binding: the B200 kernels behind attnforge's own template boundary.

``lowering.bind_executable(assemble_kernel(spec, tile), plan).run(arrays)`` (lowering.py:459-468,
850-974) is where the reference executes a lowered variant: numpy float64 arrays in, a numpy
array out.  ``B200ExecutablePlan`` is the drop-in for that object — constructed from the
reference's own ``KernelIR`` and ``ExecutionPlan`` (duck-typed: only ``ir.spec`` is read, so
attnforge need not be importable here) — and ``bind_executable`` the drop-in for the binder.
``autodiff_grads`` mirrors ``engine.autodiff_grads`` (engine.py:630-639) on numpy arrays.

Inputs are moved to the GPU as bf16 (q, k, v) / fp32 (extras), or fp32 everywhere with
``precision="fp32"`` (the exact-FFMA parallel path); outputs come back as float64 numpy.  The
tile of the reference plan does not constrain the kernels (tiled ≡ naive for any blocking,
test_engine.py:189-221).  Errors are the reference's kinds (``errors.py``).
"""

from __future__ import annotations

import numpy as np
import torch

from . import api
from .spec import Pattern, from_reference


def _to_device(spec, arrays: dict, precision: str) -> dict:
    out = {}
    for name, x in arrays.items():
        t = torch.as_tensor(np.ascontiguousarray(x), device="cuda")
        if name in ("q", "k", "v") and precision == "bf16":
            out[name] = t.to(torch.bfloat16)
        else:
            out[name] = t.to(torch.float32)
    return out


class B200ExecutablePlan:
    """``lowering.ExecutablePlan`` drop-in: ``run(arrays) -> ndarray`` on the sm_100a kernels."""

    def __init__(self, ir, plan=None, precision: str = "bf16"):
        self.ir = ir
        self.plan = plan
        self.spec = from_reference(ir.spec)
        self.precision = precision

    def run(self, arrays: dict) -> np.ndarray:
        dev = _to_device(self.spec, arrays, self.precision)
        if self.spec.pattern is Pattern.PARALLEL:
            out = api.run_tiled_parallel(self.spec, dev, precision=self.precision)
        else:
            out = api.run_chunk_recurrent(self.spec, dev)
        return out.double().cpu().numpy()


def bind_executable(ir, plan=None, precision: str = "bf16") -> B200ExecutablePlan:
    """``lowering.bind_executable`` (lowering.py:971-974) returning the B200 plan."""
    return B200ExecutablePlan(ir, plan, precision)


def autodiff_grads(spec, arrays: dict, wrt=None) -> dict:
    """``engine.autodiff_grads`` on numpy arrays: gradients of sum(O) as float64 numpy."""
    spec = from_reference(spec)
    g = api.autodiff_grads(spec, _to_device(spec, arrays, "bf16"), wrt)
    return {n: t.double().cpu().numpy() for n, t in g.items()}
