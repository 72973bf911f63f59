"""Benchmark: attention fwd+bwd TFLOPS & % of bf16 tensor peak on B200 (BASELINE.json metric).

Default workload (BASELINE.json configs[1], fits one GPU): cfg2, Llama-3 8B GQA causal softmax
attention, bf16, B=8 Hq=32 Hkv=8 S=8192 D=128 — one "step" = K1 forward (O, LSE) + K2 backward
(dQ, dK, dV) of one synthetic batch.  ``--config`` selects any other BASELINE config (cfg1, cfg3,
cfg4a, cfg4b, cfg5a, cfg5b; ``all`` prints one line per config).  Algorithmic work:

  parallel  fwd 2·B·H·P·(Dqk+Dv), bwd 2·B·H·P·(3Dqk+2Dv), P = unmasked (i, j) pairs per (b, h)
  linear    fwd B·H·S·(2c(Dk+Dv)+4·Dk·Dv) with c = 64 (lowering.py:396-399), bwd 2× fwd

  value     device-resident throughput (inputs in HBM before the timed region), TFLOPS
  e2e       the same metric through the public host-buffer API (pipeline.HostPipeline): pinned
            host inputs → H2D, kernels, D2H of every output, all inside the timed region
  roofline  dominant kernel (K2 backward, or the forward of forward-only configs): achieved
            TFLOPS ÷ measured sustained bf16 peak, or algorithmic GB/s ÷ measured HBM copy
            bandwidth for the HBM-bound configs (MLA decode, linear template)
  cpu_baseline  the float64 oracle port of the reference executors on the host cores (bounded
                sample; rank 0, N=1 only)

Multi-GPU (torchrun): every rank runs its own copy of the workload (weak scaling: batch×head units
are independent, no data-path collective); time = max over ranks.  ``--impl reference`` times the
reference's CPU algorithm (oracle port, all host cores) on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import dataclass
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "attention fwd+bwd TFLOPS & % bf16 tensor peak at 1/2/4/8 B200 vs CPU ref"
L2_BYTES = 126 * 2 ** 20

_REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                0x100: "display_clock_setting"}


@dataclass(frozen=True)
class Workload:
    key: str
    title: str
    backward: bool
    bound: str                 # "tensor" | "hbm" | "fp32-fma"
    precision: str = "bf16"
    cpu_seq: int = 1024        # sequence length of one CPU-baseline slice


WORKLOADS = {
    "cfg1": Workload("cfg1", "cfg1: causal softmax attention fwd, fp32, B1 H4 S512 D64 (the "
                     "reference's own CPU-runnable case; exact-FFMA fp32 path)", False,
                     "fp32-fma", "fp32", 512),
    "cfg2": Workload("cfg2", "cfg2: Llama-3 8B GQA causal softmax attention fwd+bwd, bf16, B8 "
                     "Hq32 Hkv8 S8192 D128", True, "tensor"),
    "cfg3": Workload("cfg3", "cfg3: sigmoid attention + relative-position score_mod + causal "
                     "sliding-window (W1024) mask_mod fwd+bwd, bf16, B8 H16 S4096 D128", True,
                     "tensor", cpu_seq=2048),
    "cfg4a": Workload("cfg4a", "cfg4a: DeepSeek-V2 MLA prefill fwd+bwd (latent KV, Dqk576 "
                      "Dv512), bf16, B1 H128 S4096 causal", True, "tensor", cpu_seq=512),
    "cfg4b": Workload("cfg4b", "cfg4b: DeepSeek-V2 MLA decode (Dqk576 Dv512), bf16, B16 H128 "
                      "Sq1 over a 32k latent KV cache", False, "hbm", cpu_seq=4096),
    "cfg5a": Workload("cfg5a", "cfg5a: RetNet retention (linear template, chunked) fwd+bwd, "
                      "bf16, B4 H16 S8192 Dk=Dv=256", True, "hbm"),
    "cfg5b": Workload("cfg5b", "cfg5b: Mamba2 SSD (linear template, chunked, differentiable "
                      "gate/decay) fwd+bwd, bf16, B4 H32 S8192 Dk=Dv=128", True, "hbm"),
}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"tflops_burst": d["bf16_tflops"], "tflops_sustained": d["bf16_tflops_sustained"],
                "hbm_gbs": d["hbm_gbs"], "source": "measured"}
    return {"tflops_burst": 1590.0, "tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
            "source": "fallback"}


# ───────────────────────────── work model ─────────────────────────────

def work(spec) -> dict:
    """Algorithmic flops and HBM bytes of one forward / backward of ``spec``."""
    from paper_2502_15349_b200 import configs
    from paper_2502_15349_b200.spec import Pattern
    d = spec.dims
    b, h, hkv = d.batch, d.heads, d.kv_heads
    if spec.pattern is Pattern.PARALLEL:
        pairs = configs.unmasked_pairs(spec)
        fwd = 2 * b * h * pairs * (d.d_qk + d.d_v)
        bwd = 2 * b * h * pairs * (3 * d.d_qk + 2 * d.d_v)
        kv = b * hkv * d.seq_k * (d.d_qk + (0 if spec.kv_shared else d.d_v)) * 2
        qo = b * h * d.seq_q * (d.d_qk + d.d_v) * 2
        fwd_bytes = kv + qo + b * h * d.seq_q * 4
        bwd_bytes = 2 * (kv + qo) + b * h * d.seq_q * (d.d_v * 2 + 4)
    else:
        c = 64
        fwd = b * h * d.seq_q * (2 * c * (d.d_qk + d.d_v) + 4 * d.d_qk * d.d_v)
        bwd = 2 * fwd
        tok = b * h * d.seq_q
        ext = sum(4 * tok for _ in spec.extra_inputs)
        fwd_bytes = tok * (2 * d.d_qk + 2 * d.d_v) * 2 + ext
        bwd_bytes = tok * (2 * d.d_qk + d.d_v) * 2 * 2 + tok * d.d_v * 2 + 2 * ext
    return {"fwd_flops": fwd, "bwd_flops": bwd, "fwd_bytes": fwd_bytes, "bwd_bytes": bwd_bytes}


def build_spec(key: str, **kw):
    from paper_2502_15349_b200 import configs
    return configs.CONFIGS[key](**kw)


# ───────────────────────────── clocks ─────────────────────────────

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for bit, name in _REASON_BITS.items():
                if bits & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ───────────────────────────── CPU baseline (the reference itself) ─────────────────────────────
# The reference is a pure-Python package: `baseline/_ref` holds it installed unmodified (pip
# --target), and the CPU legs time its own executors — engine.run_tiled_parallel /
# run_chunk_recurrent + engine.autodiff_grads (loss = sum(O)) — on (b, h) slices of the workload,
# one process per host core (parallelism over (b, h) is what the reference permits).
# Without the install the float64 oracle port (numpy matmuls, same algorithm) stands in.

REF_DIR = ROOT / "baseline" / "_ref"


def reference_available() -> bool:
    if not (REF_DIR / "attnforge" / "engine.py").exists():
        return False
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import attnforge.engine  # noqa: F401
        return True
    except Exception:  # noqa: BLE001 - a broken install falls back to the port
        return False


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cpu_sample_spec(key: str, s_len: int):
    """One (b, h) slice of the workload at a bounded sequence length."""
    w = WORKLOADS[key]
    if key == "cfg1":
        return build_spec(key)          # runs in full
    if key == "cfg2":
        return build_spec(key, batch=1, heads=1, heads_kv=1, seq=s_len)
    if key == "cfg3":
        return build_spec(key, batch=1, heads=1, seq=s_len)
    if key == "cfg4a":
        return build_spec(key, batch=1, heads=1, seq=s_len)
    if key == "cfg4b":
        return build_spec(key, batch=1, heads=8, seq_k=s_len)
    assert w.bound == "hbm"
    return build_spec(key, batch=1, heads=1, seq=s_len)


def _reference_spec(spec):
    """The same slice as an attnforge spec (variant-file dict through the reference's own
    loader).  MLA's shared latent head becomes an ordinary K/V pair of the same shapes (the
    reference has no kv_shared); a one-head slice has no GQA grouping."""
    from attnforge import variantfile as VF
    from paper_2502_15349_b200.spec import spec_to_dict
    doc = spec_to_dict(spec)
    doc.pop("kv_shared", None)
    doc["dims"].pop("heads_kv", None)
    return VF.spec_from_dict(doc)


def _cpu_slice(args):
    key, s_len, seed, kind = args
    import numpy as np
    from threadpoolctl import threadpool_limits
    from paper_2502_15349_b200.spec import Pattern
    spec = _cpu_sample_spec(key, s_len)
    w = WORKLOADS[key]
    with threadpool_limits(1):
        if kind == "reference":
            reference_available()
            from attnforge import engine as E
            rs = _reference_spec(spec)
            arrays = E.generate(rs, seed).arrays
            t0 = time.perf_counter()
            if spec.pattern is Pattern.PARALLEL:
                E.run_tiled_parallel(rs, arrays, 64, 64)
            else:
                E.run_chunk_recurrent(rs, arrays, 64)
            if w.backward:
                E.autodiff_grads(rs, arrays)
            return time.perf_counter() - t0
        import oracle
        from oracle import parallel as OP, recurrent as OR
        arrays = oracle.generate(spec, seed)
        rng = np.random.default_rng(seed)
        t0 = time.perf_counter()
        if spec.pattern is Pattern.PARALLEL:
            o = OP.tiled_forward(spec, arrays, 64, 64)
            if w.backward:
                OP.parallel_vjp(spec, arrays, rng.uniform(-1, 1, o.shape))
        else:
            o = OR.chunk_forward(spec, arrays, 64)
            if w.backward:
                OR.chunk_vjp(spec, arrays, rng.uniform(-1, 1, o.shape), chunk=64)
        return time.perf_counter() - t0


# Slice lengths of the CPU legs: the reference's autodiff holds every intermediate of the dense
# graph (≈1 GB per head at S=2048) and refuses recurrent unrolls above 256 steps
# (attention.py:475-477), so its slices are shorter than the port's.
_REF_SEQ = {"cfg1": 512, "cfg2": 1024, "cfg3": 1024, "cfg4a": 512, "cfg4b": 4096,
            "cfg5a": 256, "cfg5b": 256}


class CpuPool:
    """One spawned process per host core, imported and warmed before any timing."""

    def __init__(self, key: str, s_len: int | None, kind: str | None = None):
        import multiprocessing as mp
        self.key = key
        self.kind = kind or ("reference" if reference_available() else "port")
        self.s_len = s_len or (_REF_SEQ[key] if self.kind == "reference" else
                               WORKLOADS[key].cpu_seq)
        self.cores = 1 if key == "cfg1" else (os.cpu_count() or 1)
        self.pool = mp.get_context("spawn").Pool(self.cores)
        self.pool.map(_cpu_slice, [(key, min(self.s_len, 64) if key != "cfg1" else self.s_len,
                                    i, self.kind) for i in range(self.cores)])

    def step(self, seed0: int = 0) -> dict:
        w = WORKLOADS[self.key]
        t0 = time.perf_counter()
        self.pool.map(_cpu_slice, [(self.key, self.s_len, seed0 + i, self.kind)
                                   for i in range(self.cores)])
        wall = time.perf_counter() - t0
        sample = _cpu_sample_spec(self.key, self.s_len)
        wk = work(sample)
        flops = self.cores * (wk["fwd_flops"] + (wk["bwd_flops"] if w.backward else 0))
        if self.kind == "reference":
            what = ("engine.run_tiled_parallel(64x64)" if sample.pattern.value == "parallel"
                    else "engine.run_chunk_recurrent(64)")
            what += " + engine.autodiff_grads" if w.backward else ""
            who = "the unmodified reference (attnforge from baseline/_ref)"
        else:
            what = "fwd + VJP" if w.backward else "fwd"
            who = "the float64 oracle port (baseline/_ref absent)"
        return {"value": flops / wall / 1e12, "unit": "TFLOPS", "cores": self.cores,
                "kind": self.kind, "cpu_model": cpu_model(),
                "sample": f"{self.cores} (b,h) slice(s) of {self.key} ({sample.dims}), {what} "
                          f"by {who}, one process per core: {wall:.2f} s wall; throughput "
                          f"credits the slices' algorithmic flops",
                "wall_s": wall}

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_baseline(key: str, s_len: int | None = None) -> dict:
    pool = CpuPool(key, s_len)
    try:
        return pool.step()
    finally:
        pool.close()


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = WORKLOADS[args.config]
    pool = CpuPool(args.config, args.cpu_seq)
    try:
        for i in range(args.warmup):
            pool.step(1000 * (i + 1))
        vals, t_total = [], 0.0
        for i in range(args.steps):
            r = pool.step(i)
            vals.append(r["value"])
            t_total += r["wall_s"]
    finally:
        pool.close()
    v = statistics.median(vals)
    r["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOPS",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.title + " (CPU sample, see cpu_baseline.sample)"},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "cpu_model",
                                               "sample")},
            "e2e": {"value": v, "unit": "TFLOPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ───────────────────────────── GPU arm ─────────────────────────────

def device_inputs(spec, dev, seed: int):
    """Synthetic inputs of the workload's shapes: q/k/v uniform[-1,1] bf16 (fp32 for the fp32
    path), extras by their declared fill (unit gates 0.5+0.45·U, per-head constants)."""
    import torch
    g = torch.Generator(device=dev).manual_seed(seed)
    d = spec.dims

    def rnd(*shape, dtype=torch.bfloat16):
        return (torch.rand(*shape, device=dev, generator=g) * 2 - 1).to(dtype)

    arrays = {"q": rnd(d.batch, d.heads, d.seq_q, d.d_qk),
              "k": rnd(d.batch, d.kv_heads, d.seq_k, d.d_qk)}
    if not spec.kv_shared:
        arrays["v"] = rnd(d.batch, d.kv_heads, d.seq_k, d.d_v)
    for e in spec.extra_inputs:
        shape = e.resolve_shape(d)
        if e.fill == "unit":
            arrays[e.name] = 0.5 + 0.45 * rnd(*shape, dtype=torch.float32)
        elif e.fill == "constant_decay":
            gm = torch.tensor(e.fill_params["gamma"], device=dev, dtype=torch.float32)
            view = [1, -1, 1, 1] if shape[1] > 1 else [1, 1, 1, 1]
            arrays[e.name] = gm.reshape(view).expand(*shape).contiguous()
        else:
            arrays[e.name] = rnd(*shape, dtype=torch.float32)
    dout = rnd(d.batch, d.heads, d.seq_q, d.d_v)
    return arrays, dout


def run_gpu(args, key: str) -> dict | None:
    import torch
    import torch.distributed as dist
    import paper_2502_15349_b200 as af
    from paper_2502_15349_b200 import runtime as rt
    from paper_2502_15349_b200.pipeline import HostPipeline
    from paper_2502_15349_b200.spec import Pattern

    from paper_2502_15349_b200.shard import shard_units
    w = WORKLOADS[key]
    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    spec = build_spec(key)
    wk = work(spec)
    # Multi-GPU: the global workload is `world` copies of the config along the batch
    # axis (weak scaling); its independent units — (b, KV group) for the parallel template, (b, h)
    # for the linear one — are partitioned by shard.shard_units, which hands every rank exactly one
    # config's worth of whole batch rows.  No data-path collective runs in the timed region.
    d = spec.dims
    groups = d.kv_heads if spec.pattern is Pattern.PARALLEL else d.heads
    shard = shard_units(d.batch * world, groups, world, rank)
    b_lo = shard.units[0] // groups
    assert len(shard.units) == d.batch * groups and shard.units[0] % groups == 0, shard
    arrays, dout = device_inputs(spec, dev, 1234 + b_lo)
    if w.precision == "fp32":
        arrays = {k: v.float() for k, v in arrays.items()}
    in_bytes = sum(t.numel() * t.element_size() for t in arrays.values())
    flush = torch.empty(2 * L2_BYTES // 4, device=dev, dtype=torch.float32) \
        if in_bytes < 2 * L2_BYTES else None
    stream = torch.cuda.current_stream()
    parallel = spec.pattern is Pattern.PARALLEL

    def fwd():
        if parallel:
            return af.parallel_forward(spec, arrays, precision=w.precision)
        return af.linear_forward(spec, arrays), None

    def bwd(o, lse):
        if parallel:
            return af.parallel_backward(spec, arrays, o, lse, dout)
        return af.linear_backward(spec, arrays, dout)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        o, lse = fwd()
        if w.backward:
            bwd(o, lse)
    barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    launches0 = rt.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            ev[i][0].record(stream)
            o, lse = fwd()
            ev[i][1].record(stream)
            if w.backward:
                bwd(o, lse)
            ev[i][2].record(stream)
        barrier()
    launches = rt.launch_count() - launches0
    ms = sum(a.elapsed_time(c) for a, _, c in ev) / args.steps
    fwd_ms = sum(a.elapsed_time(b) for a, b, _ in ev) / args.steps
    bwd_ms = sum(b.elapsed_time(c) for _, b, c in ev) / args.steps
    t = torch.tensor([ms, fwd_ms, bwd_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, fwd_ms, bwd_ms = (float(x) for x in t.tolist())

    # The one collective of the path (outside the timed region): all-gather every rank's O (and
    # LSE) into the global [world*B, ...] tensors over NCCL, timed on the device, max over ranks.
    gather = None
    if world > 1:
        from paper_2502_15349_b200.shard import gather_batch_rows
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        outs = [o] + ([lse] if lse is not None else [])
        gather_batch_rows(outs, world)  # warm-up (communicator set-up)
        barrier()
        g0.record(stream)
        full = gather_batch_rows(outs, world)
        g1.record(stream)
        barrier()
        gms = torch.tensor([g0.elapsed_time(g1)], device=dev)
        dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        ok = all(torch.equal(f[b_lo: b_lo + d.batch], x) for f, x in zip(full, outs))
        nbytes = sum(x.numel() * x.element_size() for x in outs)
        gather = {"ms": float(gms.item()), "bytes_per_rank": nbytes,
                  "bus_gbs": nbytes * (world - 1) / (float(gms.item()) * 1e-3) / 1e9,
                  "what": "dist.all_gather_into_tensor of O" + (" and LSE" if lse is not None
                                                                else "") +
                          " into the global batch (NCCL), outside the timed region",
                  "own_slot_matches": bool(ok)}
        del full

    # e2e through the public host-buffer API: pinned host inputs, H2D + kernels + D2H per step
    pipe = HostPipeline(spec, device=dev, precision=w.precision)
    host = {k: v.cpu().pin_memory() for k, v in arrays.items()}
    hdo = dout.cpu().pin_memory() if w.backward else None
    out = pipe(host, hdo)
    pipe(host, hdo, out=out)  # second warm-up: the chunk streams' allocator pools are populated
    barrier()
    h2d = sum(t.numel() * t.element_size() for t in host.values()) + \
        (hdo.numel() * hdo.element_size() if hdo is not None else 0)
    d2h = sum(t.numel() * t.element_size() for t in out.values())
    e2e_steps = max(1, min(args.steps, 5))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        pipe(host, hdo, out=out)
    e1.record(stream)
    barrier()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / e2e_steps], device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    del out, host, hdo, pipe

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(key, args.cpu_seq)
        cpu.pop("wall_s", None)
    if rank != 0:
        return None

    pk = peaks()
    step_flops = wk["fwd_flops"] + (wk["bwd_flops"] if w.backward else 0)
    value = world * step_flops / (ms * 1e-3) / 1e12
    dom = "bwd" if w.backward else "fwd"
    dom_ms = bwd_ms if w.backward else fwd_ms
    traffic, traffic_src = None, None
    prof = ROOT / "profiles" / "roofline_traffic.json"
    if prof.exists():
        tdoc = json.loads(prof.read_text())
        traffic = tdoc.get(key, {}).get(f"{dom}_dram_bytes_per_launch")
        traffic_src = (f"profiles/roofline_traffic.json (ncu --set full, tag {tdoc.get('tag')}, "
                       f"head {tdoc.get('head')}): DRAM read+write bytes of the step's {dom} "
                       f"kernels")
    if w.bound == "hbm":
        achieved = wk[f"{dom}_bytes"] / (dom_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                "algorithmic_bytes": wk[f"{dom}_bytes"],
                "peak_source": f"{pk['source']} hbm_gbs"}
        if w.backward:  # the forward's share, also HBM-bound
            fa = wk["fwd_bytes"] / (fwd_ms * 1e-3) / 1e9
            roof["fwd"] = {"achieved": fa, "frac": fa / pk["hbm_gbs"]}
    elif w.bound == "tensor":
        achieved = wk[f"{dom}_flops"] / (dom_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": pk["tflops_sustained"],
                "unit": "TFLOP/s", "frac": achieved / pk["tflops_sustained"], "traffic": traffic,
                "peak_source": f"{pk['source']} bf16_tflops_sustained (the dominant kernel runs "
                               f"inside a multi-kernel step)",
                "peak_burst": pk["tflops_burst"], "frac_burst": achieved / pk["tflops_burst"]}
    else:  # exact fp32 FFMA path: nominal CUDA-core peak, 148 SMs x 128 FMA/clk x 1.965 GHz
        achieved = wk["fwd_flops"] / (fwd_ms * 1e-3) / 1e12
        peak = 148 * 128 * 2 * 1.965e9 / 1e12
        roof = {"bound": "fp32-fma", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "peak_source": "nominal fp32 FFMA (no measured figure)"}
    roof["kernel"] = {"fwd": "forward kernel(s) of the config", "bwd": "backward kernels of "
                      "the config"}[dom]
    roof["traffic_source"] = traffic_src
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if w.precision == "fp32" else "bf16",
        "data": "synthetic (uniform[-1,1] inputs, per-rank seed)",
        "config": {"workload": w.title, "global_batch": d.batch * world, "seq_len": d.seq_q,
                   "seq_k": d.seq_k, "heads_q": d.heads, "heads_kv": d.kv_heads,
                   "d_qk": d.d_qk, "d_v": d.d_v,
                   "parallelism": (f"dp{world}: batch x {'KV-group' if parallel else 'head'} "
                                   f"units partitioned by shard.shard_units, {len(shard.units)} "
                                   f"units per rank, no collective in the timed region"),
                   "l2": ("L2 flushed (2x126 MB write) before every step" if flush is not None
                          else f"inputs larger than L2 ({in_bytes / 1e6:.0f} MB per rank)")},
        "frac_of_peak": (value / world / pk["tflops_sustained"]) if w.bound == "tensor" else None,
        "fwd_ms": fwd_ms, "bwd_ms": bwd_ms if w.backward else None,
        "fwd_tflops": wk["fwd_flops"] / (fwd_ms * 1e-3) / 1e12,
        "bwd_tflops": wk["bwd_flops"] / (bwd_ms * 1e-3) / 1e12 if w.backward else None,
        "tokens_per_s": world * d.batch * d.seq_q / (ms * 1e-3),
        "e2e": {"value": world * step_flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOPS",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "api": "paper_2502_15349_b200.pipeline.HostPipeline (pinned host tensors; H2D, "
                       "kernels and D2H overlapped over batch/KV-head chunks)"},
        "roofline": roof,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if gather is not None:
        line["gather"] = gather
    return line


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(WORKLOADS) + ["all"], default="cfg2")
    ap.add_argument("--cpu-seq", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 untimed warm-up steps
    keys = sorted(WORKLOADS) if args.config == "all" else [args.config]
    if len(keys) > 1 and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        # one fresh process per config, so no config inherits another's allocator / host state
        for k in keys:
            cmd = [sys.executable, str(Path(__file__).resolve()), "--config", k, "--impl",
                   args.impl, "--steps", str(args.steps), "--warmup", str(args.warmup),
                   "--gpus", str(args.gpus)]
            if args.cpu_seq is not None:
                cmd += ["--cpu-seq", str(args.cpu_seq)]
            if args.no_cpu:
                cmd.append("--no-cpu")
            subprocess.run(cmd, check=False)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (the driver's own launch
        # sets WORLD_SIZE and lands below directly)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        sys.exit(subprocess.run(cmd, env=env).returncode)
    if args.impl == "reference":
        for k in keys:
            args.config = k
            run_reference(args)
        return
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    for k in keys:
        line = run_gpu(args, k)
        if line is not None:
            print(json.dumps(line), flush=True)
        torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
