"""Developer probe: run the cfg4b decode step many times (hang / determinism check)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402

spec = bench.build_spec(sys.argv[1] if len(sys.argv) > 1 else "cfg4b")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
arrays, _ = bench.device_inputs(spec, torch.device("cuda"), 0)
o0, l0 = af.parallel_forward(spec, arrays)
torch.cuda.synchronize()
bad = 0
for i in range(reps):
    o, l = af.parallel_forward(spec, arrays)
    torch.cuda.synchronize()
    bad += int(not (torch.equal(o, o0) and torch.equal(l, l0)))
    print(i, flush=True) if i % 10 == 0 else None
print(f"{reps} runs, {bad} differ from the first", flush=True)
