"""Developer timeline of one K2f (fused backward) CTA at cfg2 (build with
AF_EXTRA_NVCC_FLAGS=-DAF_FUSED_TRACE): per-iteration event times relative to the row warps'
s_full, averaged over the steady state, and the iteration period."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import runtime as rt  # noqa: E402

spec = bench.build_spec(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
for _ in range(2):
    o, lse = af.parallel_forward(spec, arrays)
    af.parallel_backward(spec, arrays, o, lse, dout)
torch.cuda.synchronize()
buf = np.zeros((16, 512), dtype=np.int64)
fn = rt.lib().af_debug_fused_trace
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p]
assert fn(buf.ctypes.data) == 0
names = {0: "mma: p_ready(n) passed", 1: "mma: dP(n) issued", 2: "mma: ds_ready(n) passed",
         3: "mma: S(n) issued", 4: "rows: s_full(n) passed", 5: "rows: p_ready(n) arrived",
         6: "rows: dp_full(n) passed", 7: "rows: ds_free(n-2) passed",
         8: "rows: ds_ready(n) arrived", 9: "drain: dq_full(n) passed",
         10: "drain: dq_free(n) arrived", 12: "tma: Q/dO(n) issued"}
nk = int((buf[4] > 0).sum())
ss = range(8, max(9, nk - 8))
base = buf[4]
print(f"iterations traced {nk}; period (rows s_full to s_full): "
      f"{np.mean([buf[4, n + 1] - buf[4, n] for n in ss]):.0f} clk")
rel = {e: np.mean([buf[e, n] - base[n] for n in ss]) for e in names}
for e in sorted(names, key=lambda e: rel[e]):
    print(f"  {names[e]:30s} {rel[e]:8.0f}")
