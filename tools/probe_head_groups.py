"""Developer probe: cfg4a backward time vs the materialised backward's head-chunk count
(schedule.Candidate(head_groups=g); 0 = the default formula)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import schedule  # noqa: E402

spec = bench.build_spec(sys.argv[1] if len(sys.argv) > 1 else "cfg4a")
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
o, lse = af.parallel_forward(spec, arrays)
for g in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0,8,16,24,32,48,64".split(","))]:
    schedule.clear()
    if g:
        schedule.record(spec, schedule.Candidate(head_groups=g))
    for _ in range(2):
        af.parallel_backward(spec, arrays, o, lse, dout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        af.parallel_backward(spec, arrays, o, lse, dout)
    e1.record()
    torch.cuda.synchronize()
    print(f"head_groups {g:3d}: backward {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
schedule.clear()
