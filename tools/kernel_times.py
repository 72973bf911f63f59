"""Developer probe: per-kernel device time of one config's step, averaged over warm steps, from the
CUDA activity trace of torch.profiler (kernels run back to back as in the bench, unlike ncu's
serialised replay).  Usage: python tools/kernel_times.py cfg4a [steps]"""
import sys
from collections import defaultdict
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = bench.WORKLOADS[key]
spec = bench.build_spec(key)
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
par = spec.pattern.value == "parallel"


def step():
    if par:
        o, lse = af.parallel_forward(spec, arrays, precision=w.precision)
        if w.backward:
            af.parallel_backward(spec, arrays, o, lse, dout)
    else:
        af.linear_forward(spec, arrays)
        if w.backward:
            af.linear_backward(spec, arrays, dout)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name == "CUDA":
        a = agg[e.name[:90]]
        a[0] += 1
        a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
total = sum(t for _, t in agg.values())
print(f"{key}: {total / steps / 1e3:.3f} ms of kernels per step")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {t / steps / 1e3:8.3f} ms  x{n // steps:<3d} {name}")
