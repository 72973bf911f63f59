"""Small forward + backward launches of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): tools/sanitize.sh runs this under each tool."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import configs  # noqa: E402

dev = torch.device("cuda")
cases = {
    "K1/K2f softmax GQA causal": configs.cfg2(batch=1, heads=4, heads_kv=2, seq=384),
    "K1/K2 sigmoid relpos SWA": configs.cfg3(batch=1, heads=2, seq=512, window=200),
    "K3/K3b MLA prefill": configs.cfg4a(heads=2, seq=256),
    "K3 MLA decode": configs.cfg4b(batch=2, seq_k=1024),
    "K4/K5 RetNet 256": configs.cfg5a(batch=1, heads=1, seq=300),
    "K4/K5 Mamba2 128": configs.cfg5b(batch=1, heads=2, seq=300),
    "materialised tier (256/512)": af.builtin("retention-parallel", batch=1, heads=1, seq=64),
    "K2a/K2b split (deterministic) backward": configs.cfg2(batch=1, heads=4, heads_kv=2, seq=384),
    # the materialised backward's separate-K/V form on CTA pairs (dK pair GEMM N = 128, dV 256)
    "K3b softmax-diff 128/256": af.with_causal_mask(af.builtin(
        "softmax-diff", batch=1, heads=2, seq=300, d_qk=128, d_v=256)),
}
only = sys.argv[1:]  # case indices (default: all)
for idx, (name, spec) in enumerate(cases.items()):
    if only and str(idx) not in only:
        continue
    af.api.use_deterministic_backward(name.startswith("K2a/K2b"))
    arrays, dout = bench.device_inputs(spec, dev, 0)
    if spec.pattern.value == "parallel":
        o, lse = af.parallel_forward(spec, arrays)
        if spec.dims.seq_q > 1:
            af.parallel_backward(spec, arrays, o, lse, dout)
    else:
        af.linear_forward(spec, arrays)
        af.linear_backward(spec, arrays, dout)
    torch.cuda.synchronize()
    print("ok", name, flush=True)
