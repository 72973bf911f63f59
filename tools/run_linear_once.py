"""Run the linear template once (forward, or forward + backward) at a BASELINE config — the
target of ncu captures (`ncu ... python tools/run_linear_once.py cfg5b [bwd]`)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg5b"
spec = bench.build_spec(key)
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
for _ in range(2):
    af.linear_forward(spec, arrays)
    if len(sys.argv) > 2 and sys.argv[2] == "bwd":
        af.linear_backward(spec, arrays, dout)
torch.cuda.synchronize()
