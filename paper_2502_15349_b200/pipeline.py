"""Host-buffer executor: H2D copy, kernels and D2H copy overlapped over independent units.

The reference's callers hand the executors host arrays and read host arrays back
(``engine.run_tiled_parallel`` / ``autodiff_grads``, engine.py:423, 630).  On a B200 the naive
translation — copy everything in, compute, copy everything out — serialises two PCIe transfers
with the kernels.  Batch × KV-head units are independent, so this executor splits the
work into unit chunks and runs three CUDA streams:

    h2d  : copy chunk c+1's inputs (pinned host → a device slot)
    comp : K1 forward + K2 backward (or K4/K5) on chunk c
    d2h  : copy chunk c-1's outputs back into the caller's pinned host tensors

Host→device and device→host use separate copy engines, so in steady state the step costs
max(H2D, kernels, D2H) per chunk instead of their sum.  Device input and output slots are
double-buffered and persistent across calls (``api.reuse_buffers``): chunk c+2 writes slot
c % 2 only after chunk c's inputs are consumed and its outputs copied out.
The call is stream-ordered with the caller's current stream on both ends (its events bracket the
whole pipeline).
"""

from __future__ import annotations

from dataclasses import replace

import torch

from . import api
from .errors import InputError
from .plan import plan_linear, plan_parallel
from .spec import AttentionSpec, Pattern


# unit = (mode, b, lo, hi): mode _BATCH is the batch range [lo, hi); _KV_GROUP the KV-head group
# range [lo, hi) of batch element b (with its query heads); _HEADS_SHARED_KV the query-head range
# [lo, hi) of batch element 0 with the shared latent KV (MLA) copied whole and its gradient summed
# over the chunks
_BATCH, _KV_GROUP, _HEADS_SHARED_KV = -1, 0, 1


def _ranges(n_items: int, n: int) -> list[tuple[int, int]]:
    bounds = [round(i * n_items / n) for i in range(n + 1)]
    return [(bounds[i], bounds[i + 1]) for i in range(n)]


def _chunks(spec: AttentionSpec, max_chunks: int) -> list[tuple[int, int, int, int]]:
    """Batch ranges when B ≥ max_chunks; else (batch, KV-head group) units so that small batches
    still fill the pipeline (its fill / drain is one chunk's copies); query-head ranges when one
    latent KV head is shared by all heads (MLA, B = 1)."""
    d = spec.dims
    if d.batch >= max_chunks or (d.batch > 1 and d.kv_heads == 1):
        return [(_BATCH, 0, lo, hi) for lo, hi in _ranges(d.batch, min(max_chunks, d.batch))]
    if d.batch == 1 and spec.kv_shared and d.kv_heads == 1 and d.heads > 1:
        return [(_HEADS_SHARED_KV, 0, lo, hi)
                for lo, hi in _ranges(d.heads, min(max_chunks, d.heads))]
    per_b = min(d.kv_heads, max(1, round(max_chunks / d.batch)))
    return [(_KV_GROUP, b, lo, hi) for b in range(d.batch)
            for lo, hi in _ranges(d.kv_heads, per_b)]


def _sub_spec(spec: AttentionSpec, unit) -> AttentionSpec:
    mode, _, lo, hi = unit
    d = spec.dims
    if mode == _BATCH:
        return replace(spec, dims=replace(d, batch=hi - lo))
    if mode == _HEADS_SHARED_KV:
        return replace(spec, dims=replace(d, heads=hi - lo))
    r = d.heads // d.kv_heads
    heads_kv = None if d.heads_kv is None else hi - lo
    return replace(spec, dims=replace(d, batch=1, heads=(hi - lo) * r, heads_kv=heads_kv))


def _slice(t: torch.Tensor, spec: AttentionSpec, unit, kv: bool) -> torch.Tensor:
    """Slice a [B|1, H|1, ...] host tensor to one unit chunk."""
    mode, b, lo, hi = unit
    d = spec.dims
    if mode == _BATCH:
        return t[lo:hi] if t.shape[0] > 1 else t
    if mode == _HEADS_SHARED_KV:
        return t if kv or t.shape[1] == 1 else t[:, lo:hi]
    r = 1 if kv else d.heads // d.kv_heads
    t = t[b:b + 1] if t.shape[0] > 1 else t
    return t[:, lo * r: hi * r] if t.shape[1] > 1 else t


def _same_lowering(spec: AttentionSpec, sub: AttentionSpec) -> bool:
    """A hook that reads the ``batch``/``heads`` constants would change meaning in a chunk."""
    if spec.pattern is Pattern.PARALLEL:
        a, b = plan_parallel(spec), plan_parallel(sub)
        return (a.family, a.act, a.scale, a.bias, a.slope_const, a.band) == \
               (b.family, b.act, b.scale, b.bias, b.slope_const, b.band)
    a, b = plan_linear(spec), plan_linear(sub)
    return (a.q_scale, a.decay_const) == (b.q_scale, b.decay_const)


class HostPipeline:
    """``HostPipeline(spec)(host_arrays, host_dout=None)`` → dict of pinned host tensors.

    Forward only (``host_dout is None``): ``{"o", "lse"?}``.  Forward + backward: also the
    gradients ``{"q", "k", "v"?, ...}`` exactly as ``parallel_backward`` / ``linear_backward``
    return them.  ``out`` may pass preallocated pinned host tensors (same keys) to avoid
    allocating pinned memory per call."""

    def __init__(self, spec, device=None, max_chunks: int = 16, precision: str = "bf16",
                 overlap_calls: bool = True):
        self.spec = api._spec(spec)
        self.precision = precision
        self.device = (torch.device("cuda", torch.cuda.current_device()) if device is None
                       else torch.device(device))
        units = _chunks(self.spec, max_chunks)
        if len(units) > 1 and not _same_lowering(self.spec, _sub_spec(self.spec, units[0])):
            units = [(_BATCH, 0, 0, self.spec.dims.batch)]  # one chunk: the spec itself
        self.units = units
        # gradients of the shared latent KV: per-chunk partials summed on the device
        self._summed = {"k"} if units[0][0] == _HEADS_SHARED_KV else set()
        self._acc: dict = {}
        self.h2d = torch.cuda.Stream(self.device)
        self.comp = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self._slots: list[dict] = [{}, {}]
        self._obufs: list[dict] = [{}, {}]  # per-slot output / workspace buffers (api reuse)
        # the last call's final use of each slot: the next call's first chunks wait on these
        # rather than on the caller stream, so consecutive calls overlap (call N+1's H2D runs
        # under call N's last kernels and D2H copies instead of after them)
        self._prev_comp_done: list = [None, None]
        self._prev_out_read: list = [None, None]
        self.overlap_calls = overlap_calls  # False: every call starts after the caller's work

    # device slot tensor for one host slice (reused across calls of the same shape)
    def _slot(self, s: int, name: str, like: torch.Tensor) -> torch.Tensor:
        key = (name, tuple(like.shape), like.dtype)  # ramp units of several widths coexist
        t = self._slots[s].get(key)
        if t is None:
            with torch.cuda.stream(self.h2d):
                t = torch.empty(like.shape, dtype=like.dtype, device=self.device)
            self._slots[s][key] = t
        return t

    def _outputs_like(self, dev_out: dict) -> dict:
        d = self.spec.dims
        out = {}
        for name, t in dev_out.items():
            if t is None:
                continue
            shape = list(t.shape)
            if self.units[0][0] == _BATCH:
                shape[0] = d.batch
            elif self.units[0][0] == _HEADS_SHARED_KV:
                if name not in self._summed:
                    shape[1] = d.heads
            else:
                kv = name in ("k", "v") and d.heads_kv is not None
                shape[0] = d.batch
                shape[1] = d.kv_heads if kv else d.heads
            out[name] = torch.empty(shape, dtype=t.dtype).pin_memory()
        return out

    def _run_unit(self, arrays: dict, dout):
        spec = self._unit_spec
        if spec.pattern is Pattern.PARALLEL:
            o, lse = api.parallel_forward(spec, arrays, precision=self.precision)
            res = {"o": o, "lse": lse}
            if dout is not None:
                res.update(api.parallel_backward(spec, arrays, o, lse, dout))
        else:
            o = api.linear_forward(spec, arrays)
            res = {"o": o}
            if dout is not None:
                res.update(api.linear_backward(spec, arrays, dout))
        return res

    def __call__(self, host_arrays: dict, host_dout=None, out: dict | None = None) -> dict:
        for name, t in list(host_arrays.items()) + ([("dout", host_dout)] if host_dout is not
                                                    None else []):
            if not isinstance(t, torch.Tensor) or t.is_cuda:
                raise InputError("HostPipeline takes host tensors", name=name)
        caller = torch.cuda.current_stream(self.device)
        # (no wait on the caller stream: the inputs are host memory, and the device buffers this
        # call reuses are guarded by the previous call's per-slot events below)
        if not self.overlap_calls:
            start = torch.cuda.Event()
            start.record(caller)
            for st in (self.h2d, self.comp, self.d2h):
                st.wait_event(start)
        kv_names = {"k", "v"}
        in_ready = [torch.cuda.Event() for _ in self.units]
        comp_done = [torch.cuda.Event() for _ in self.units]
        out_read = [torch.cuda.Event() for _ in self.units]
        host_out = out
        for c, unit in enumerate(self.units):
            s = c % 2
            self._unit_spec = _sub_spec(self.spec, unit)
            if c >= 2:
                self.h2d.wait_event(comp_done[c - 2])  # slot s inputs no longer read
            elif self._prev_comp_done[s] is not None:
                self.h2d.wait_event(self._prev_comp_done[s])
            dev = {}
            with torch.cuda.stream(self.h2d):
                for name, t in host_arrays.items():
                    if name in ("qidx", "kidx"):
                        continue
                    hs = _slice(t, self.spec, unit, name in kv_names)
                    dt = self._slot(s, name, hs)
                    dt.copy_(hs, non_blocking=True)
                    dev[name] = dt
                ddo = None
                if host_dout is not None:
                    hs = _slice(host_dout, self.spec, unit, False)
                    ddo = self._slot(s, "dout", hs)
                    ddo.copy_(hs, non_blocking=True)
                in_ready[c].record(self.h2d)
            self.comp.wait_event(in_ready[c])
            if c >= 2:
                self.comp.wait_event(out_read[c - 2])  # slot s outputs copied out
            elif self._prev_out_read[s] is not None:
                self.comp.wait_event(self._prev_out_read[s])
            # outputs and workspaces come from the slot's persistent buffers: no per-chunk
            # allocation on the host path (fresh 100 MB-class allocations per chunk made the
            # enqueue, not the copies, the bound)
            with torch.cuda.stream(self.comp), api.reuse_buffers(self._obufs[s]):
                res = self._run_unit(dev, ddo)
                for name in self._summed & res.keys():
                    acc = self._acc.get(name)
                    if acc is None or acc.shape != res[name].shape:
                        acc = self._acc[name] = torch.empty(res[name].shape, dtype=torch.float32,
                                                            device=self.device)
                    if c == 0:
                        acc.copy_(res[name])
                    else:
                        acc.add_(res[name])
                comp_done[c].record(self.comp)
            if host_out is None:
                host_out = self._outputs_like(res)
            self.d2h.wait_event(comp_done[c])
            with torch.cuda.stream(self.d2h):
                for name, t in res.items():
                    if t is None or name in self._summed:
                        continue
                    t.record_stream(self.d2h)
                    _slice(host_out[name], self.spec, unit, name in kv_names and
                           self.spec.dims.heads_kv is not None).copy_(t, non_blocking=True)
                out_read[c].record(self.d2h)
        if self._summed & res.keys():
            with torch.cuda.stream(self.comp):
                summed = {n: self._acc[n].to(host_out[n].dtype) for n in self._summed & res.keys()}
                done = torch.cuda.Event()
                done.record(self.comp)
            self.d2h.wait_event(done)
            with torch.cuda.stream(self.d2h):
                for n, t in summed.items():
                    t.record_stream(self.d2h)
                    host_out[n].copy_(t, non_blocking=True)
        n = len(self.units)
        for c in range(max(0, n - 2), n):
            self._prev_comp_done[c % 2] = comp_done[c]
            self._prev_out_read[c % 2] = out_read[c]
        end = torch.cuda.Event()
        end.record(self.d2h)
        caller.wait_event(end)
        return host_out
