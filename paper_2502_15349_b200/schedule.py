"""Measured tile scheduling on the B200.

The reference chooses a tile configuration per variant with an exhaustive search scored by an
analytic cost model, or — ``attnforge schedule --mode measured`` — by timing every candidate
(``commands._measure_factory``, commands.py:200-219, feeding ``scheduling.profile(mode=
"measured")``, scheduling.py:256-266, through ``tile_config_scheduling``, 288-313).  Here the
candidates are the sm_100a kernels' runtime-selectable tile configurations and ``measure`` runs
the real kernels on the GPU (CUDA events, median of a few launches after a warm-up):

  parallel, fused softmax / sigmoid, head dims <= 128   K1 K/V ring depth   kv_stages in {2, 1}
  MLA decode (576 / 512, seq_q = 1)                   KV splits           splits in {auto, ...}
  materialised backward (MLA, 192/128, 128/256)        head groups         head_groups in {...}

``tile_config_scheduling(task, mode="measured")`` returns the fastest candidate (ties: the
earlier, i.e. the library default) and records it; ``api`` launches then use the recorded choice
for that spec (``tuning(spec)``).  ``mode="analytic"`` returns the library defaults with the flop
model's cost at the measured peak (no GPU work).
"""

from __future__ import annotations

import json
import statistics
from dataclasses import dataclass, field
from pathlib import Path

from .spec import AttentionSpec, Pattern

# recorded choices: spec repr -> tuning dict (applied by api.py to every launch of that spec)
_CHOSEN: dict[str, dict] = {}


@dataclass(frozen=True)
class Candidate:
    """One tile configuration: descriptor fields (0 = library default)."""

    kv_stages: int = 0
    splits: int = 0
    head_groups: int = 0

    def as_dict(self) -> dict:
        return {"kv_stages": self.kv_stages, "splits": self.splits,
                "head_groups": self.head_groups}


@dataclass
class SchedulingTask:
    """``lowering.make_scheduling_task`` analogue (lowering.py:362-407): the spec, its flop count
    and the candidate set; ``measure(candidate) -> seconds`` when measured mode is available."""

    name: str
    spec: AttentionSpec
    flops: float
    candidates: list = field(default_factory=list)
    measure: object = None
    kind: str = ""


@dataclass(frozen=True)
class ExecutionPlan:
    """The chosen configuration and its cost (seconds), ``scheduling.ExecutionPlan``'s role."""

    candidate: Candidate
    cost: float
    mode: str
    costs: tuple = ()


def _key(spec: AttentionSpec) -> str:
    return repr(spec)


def tuning(spec: AttentionSpec) -> dict:
    """The recorded tile configuration of ``spec`` (empty: library defaults)."""
    return _CHOSEN.get(_key(spec), {})


def record(spec: AttentionSpec, cand: Candidate) -> None:
    _CHOSEN[_key(spec)] = cand.as_dict()


def clear() -> None:
    _CHOSEN.clear()


def make_scheduling_task(spec: AttentionSpec, measure=None) -> SchedulingTask:
    from .api import MLA_DQK, MLA_DV, route_parallel
    d = spec.dims
    if spec.pattern is not Pattern.PARALLEL:
        flops = float(d.batch * d.heads * d.seq_q * (2 * 64 * (d.d_qk + d.d_v)
                                                     + 4 * d.d_qk * d.d_v))
        return SchedulingTask(spec.name, spec, flops, [Candidate()], measure, "linear")
    flops = float(2 * d.batch * d.heads * d.seq_q * d.seq_k * (d.d_qk + d.d_v))
    route, plan = route_parallel(spec)
    cands = [Candidate()]
    kind = route
    if route == "fused":
        mla = spec.kv_shared and (d.d_qk, d.d_v) == (MLA_DQK, MLA_DV)
        if mla and d.seq_q == 1:
            kind = "mla-decode"
            blocks = (d.seq_k + 31) // 32
            cands += [Candidate(splits=s) for s in (2, 4, 6, 8, 9, 12, 16, 24, 32) if s <= blocks]
        elif mla or (d.d_qk, d.d_v) in ((192, 128), (128, 256)):
            kind = "materialised-bwd"
            cands += [Candidate(head_groups=g) for g in (1, 2, 4, 8, 16) if g <= d.heads]
        elif max(d.d_qk, d.d_v) <= 128:
            kind = "k1"
            cands.append(Candidate(kv_stages=1))
    return SchedulingTask(spec.name, spec, flops, cands, measure, kind)


def measure_factory(spec: AttentionSpec, seed: int = 0, reps: int = 5):
    """``commands._measure_factory`` for the B200: synthetic inputs of the spec's shapes on
    cuda (uniform[-1, 1] bf16, extras by their fill), one timed forward (+ backward for the
    materialised-backward candidates) per call, CUDA events, median over ``reps``."""
    import torch

    from . import api
    d = spec.dims
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(seed)

    def rnd(*shape, dtype=torch.bfloat16):
        return (torch.rand(*shape, device=dev, generator=g) * 2 - 1).to(dtype)

    arrays = {"q": rnd(d.batch, d.heads, d.seq_q, d.d_qk),
              "k": rnd(d.batch, d.kv_heads, d.seq_k, d.d_qk)}
    if not spec.kv_shared:
        arrays["v"] = rnd(d.batch, d.kv_heads, d.seq_k, d.d_v)
    for e in spec.extra_inputs:
        shape = e.resolve_shape(d)
        if e.fill == "constant_decay":
            gm = torch.tensor(e.fill_params["gamma"], device=dev, dtype=torch.float32)
            arrays[e.name] = gm.reshape([1, -1, 1, 1] if shape[1] > 1 else [1, 1, 1, 1]).expand(
                *shape).contiguous()
        else:
            arrays[e.name] = 0.5 + 0.45 * rnd(*shape, dtype=torch.float32)
    dout = rnd(d.batch, d.heads, d.seq_q, d.d_v)
    task = make_scheduling_task(spec)
    with_bwd = task.kind == "materialised-bwd"

    def run(cand: Candidate):
        with api.tuned(cand.as_dict()):
            o, lse = api.parallel_forward(spec, arrays)
            if with_bwd:
                api.parallel_backward(spec, arrays, o, lse, dout)

    def measure(cand: Candidate) -> float:
        run(cand)  # warm-up (module load, tensor maps, allocator)
        times = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(cand)
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3)
        return statistics.median(times)

    return measure


def tile_config_scheduling(task: SchedulingTask, device=None, mode: str = "analytic",
                          remember: bool = True) -> ExecutionPlan:
    """``scheduling.tile_config_scheduling`` (scheduling.py:288-313): every candidate is profiled
    and the minimum returned, ordered by (cost, candidate index) so ties keep the default."""
    from .errors import InputError, UnsupportedError
    if mode == "analytic":
        peak = _peak_tflops() * 1e12
        return ExecutionPlan(task.candidates[0], task.flops / peak, mode,
                             (task.flops / peak,))
    if mode != "measured":
        raise InputError("unknown profiling mode", mode=mode)
    if task.measure is None:
        raise UnsupportedError("measured profiling unavailable for this task",
                               kind="mode-measured-unavailable", task=task.name)
    costs = [float(task.measure(c)) for c in task.candidates]
    best = min(range(len(costs)), key=lambda i: (costs[i], i))
    plan = ExecutionPlan(task.candidates[best], costs[best], mode, tuple(costs))
    if remember:
        record(task.spec, plan.candidate)
    return plan


def schedule(spec: AttentionSpec, mode: str = "measured", seed: int = 0) -> dict:
    """``commands.cmd_schedule`` payload shape (commands.py:222-262) for the B200 kernels."""
    task = make_scheduling_task(spec, measure_factory(spec, seed) if mode == "measured" else None)
    plan = tile_config_scheduling(task, mode=mode)
    return {"variant": spec.name, "device": "B200 (sm_100a)", "mode": mode, "kind": task.kind,
            "plan": plan.candidate.as_dict(), "cost": plan.cost,
            "candidates": [{"config": c.as_dict(), "cost": x}
                           for c, x in zip(task.candidates, plan.costs)]}


def _peak_tflops() -> float:
    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["bf16_tflops_sustained"])
        except (KeyError, ValueError):
            pass
    return 1400.0
