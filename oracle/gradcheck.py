"""Central finite-difference check of the oracle's closed-form VJPs (TEST INFRASTRUCTURE).

Restates attnforge ``engine.finite_diff_check`` (engine.py:651-706, policy
docs/gradcheck-policy.md): every probed coordinate evaluates loss = sum(dout * O) at x ± eps with
the oracle's float64 forward, fd = (L+ − L−) / 2eps, and compares it with the oracle VJP
(``parallel.parallel_vjp`` / ``recurrent.chunk_vjp``) through
rel err = |ad − fd| / max(1, |fd|, |ad|).  A coordinate whose two perturbed runs take different
branches is a kink and is excluded (engine.py:692-694).  The reference detects branches through
its graph's branch signature; here the signature is the sign pattern of the final scores and the
abssum clamp pattern (parallel template) or of the pre-modified q/k/v (recurrent template) —
the only non-smooth points of the hooks the oracle's closed forms cover.  Exhaustive mode
(``sample_per_tensor=None``) excludes kinks; sampled mode refills from a seeded permutation.

Only ``tests/`` import this module; the product package never does.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import parallel as OP
from . import recurrent as OR


@dataclass
class GradReport:
    name: str
    checked: int
    excluded: int
    max_rel_err: float
    worst_coord: tuple | None


def _is_parallel(spec) -> bool:
    return spec.pattern.name == "PARALLEL"


def _forward(spec, arrays):
    if _is_parallel(spec):
        return OP.naive_forward(spec, arrays)
    return OR.step_forward(spec, arrays)


def _signature(spec, arrays) -> bytes:
    with np.errstate(all="ignore"):
        if _is_parallel(spec):
            _, _, _, _, z, _ = OP.final_scores(spec, arrays)
            zf = np.where(np.isfinite(z), z, 0.0)
            parts = [np.signbit(zf), zf == 0.0, np.isfinite(z)]
            if OP._classify(spec) == "abssum":
                parts.append(np.sum(np.abs(zf), -1) >= 1.0)
        else:
            parts = [np.signbit(x) for x in OR._premod(spec, arrays)]
    return b"".join(np.packbits(np.asarray(p, bool)).tobytes() for p in parts)


def _vjp(spec, arrays, dout):
    if _is_parallel(spec):
        return OP.parallel_vjp(spec, arrays, dout)
    return OR.chunk_vjp(spec, arrays, dout, chunk=max(1, spec.dims.seq_q // 3))


def finite_diff_check(spec, arrays: dict, wrt=None, eps: float = 1e-5, rel_tol: float = 1e-5,
                      sample_per_tensor: int | None = None, seed: int = 0, dout=None):
    """(ok, [GradReport]) — engine.finite_diff_check's contract (engine.py:651-706) applied to the
    oracle.  ``dout`` defaults to ones (loss = sum(O), the reference's seed)."""
    arrays = {k: np.array(v, np.float64, copy=True) for k, v in arrays.items()}
    o = _forward(spec, arrays)
    dout = np.ones_like(o) if dout is None else np.asarray(dout, np.float64)
    ad = _vjp(spec, arrays, dout)
    if wrt is None:
        wrt = [n for n in ad if n in ("q", "k", "v") or any(
            e.name == n and e.differentiable for e in spec.extra_inputs)]
    reports, ok = [], True
    for ti, name in enumerate(wrt):
        grad, arr = ad[name], arrays[name]
        coords = list(np.ndindex(arr.shape))
        quota = None
        if sample_per_tensor is not None and len(coords) > sample_per_tensor:
            perm = np.random.default_rng((seed << 16) + 9000 + ti).permutation(len(coords))
            coords = [coords[i] for i in perm]
            quota = sample_per_tensor
        checked = excluded = 0
        max_err, worst = 0.0, None
        for coord in coords:
            if quota is not None and checked >= quota:
                break
            base = arr[coord]
            arr[coord] = base + eps
            sp, lp = _signature(spec, arrays), float(np.sum(dout * _forward(spec, arrays)))
            arr[coord] = base - eps
            sm, lm = _signature(spec, arrays), float(np.sum(dout * _forward(spec, arrays)))
            arr[coord] = base
            if sp != sm:
                excluded += 1
                continue
            fd = (lp - lm) / (2.0 * eps)
            a = float(grad[coord])
            err = abs(a - fd) / max(1.0, abs(fd), abs(a))
            checked += 1
            if err > max_err:
                max_err, worst = err, coord
        if max_err > rel_tol:
            ok = False
        reports.append(GradReport(name, checked, excluded, max_err, worst))
    return ok, reports
