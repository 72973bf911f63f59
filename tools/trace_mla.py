"""Developer timeline of one MLA prefill CTA (build with AF_EXTRA_NVCC_FLAGS=-DAF_MLA_TRACE)."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import runtime as rt  # noqa: E402

spec = bench.build_spec(sys.argv[1] if len(sys.argv) > 1 else "cfg4a")
arrays, _ = bench.device_inputs(spec, torch.device("cuda"), 0)
for _ in range(3):
    af.parallel_forward(spec, arrays)
torch.cuda.synchronize()
buf = np.zeros((10, 128), dtype=np.int64)
fn = rt.lib().af_debug_mla_trace
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p]
assert fn(buf.ctypes.data) == 0
names = ["tma: k_empty passed", "mma: k_full passed (S issue)", "mma: p_ready passed (PV issue)",
         "softmax: s_full passed", "softmax: P published", "softmax: S loaded",
         "softmax: max done", "softmax: exps done", "softmax: P stored"]
ss = range(8, 56) if (buf[3] > 0).sum() > 60 else range(4, int((buf[3] > 0).sum()) - 2)
base = buf[3]
print(f"period (softmax s_full to s_full): {np.mean([buf[3, n + 1] - buf[3, n] for n in ss]):.0f}")
for e in np.argsort([np.mean([buf[e, n] - base[n] for n in ss]) for e in range(9)]):
    print(f"  {names[e]:32s} {np.mean([buf[e, n] - base[n] for n in ss]):8.0f}")
