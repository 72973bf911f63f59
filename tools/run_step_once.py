"""One step (forward, + backward where the config has one) of a BASELINE config with the bench's
own synthetic inputs — the target of the ncu captures behind profiles/ (no warm-up: ncu replays
each kernel with caches flushed, so the first step's launches are representative)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = bench.WORKLOADS[key]
spec = bench.build_spec(key)
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
if w.precision == "fp32":
    arrays = {k: v.float() for k, v in arrays.items()}
if spec.pattern.value == "parallel":
    o, lse = af.parallel_forward(spec, arrays, precision=w.precision)
    if w.backward:
        af.parallel_backward(spec, arrays, o, lse, dout)
else:
    af.linear_forward(spec, arrays)
    if w.backward:
        af.linear_backward(spec, arrays, dout)
torch.cuda.synchronize()
