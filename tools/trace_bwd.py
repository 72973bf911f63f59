"""Developer timeline of one K2b (dQ) CTA at cfg2 (build with AF_EXTRA_NVCC_FLAGS=-DAF_BWD_TRACE)."""
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
buf = np.zeros((10, 256), dtype=np.int64)
fn = rt.lib().af_debug_bwd_trace
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p]
assert fn(buf.ctypes.data) == 0
names = ["mma: ds_ready[0] passed", "mma: ds_ready[1] passed", "mma: S/dP(n+1, 0) issued",
         "mma: S/dP(n+1, 1) issued", "rows0: s_full passed", "rows1: s_full passed",
         "rows0: dp_full passed", "rows1: dp_full passed", "rows0: dS published",
         "rows1: dS published"]
nk = int((buf[4] > 0).sum())
ss = range(8, max(9, nk - 8))
base = buf[4]
print(f"tiles traced {nk}; period (rows0 s_full to s_full): "
      f"{np.mean([buf[4, n + 1] - buf[4, n] for n in ss]):.0f} clk")
order = sorted(range(10), key=lambda e: np.mean([buf[e, n] - base[n] for n in ss]))
for e in order:
    print(f"  {names[e]:28s} {np.mean([buf[e, n] - base[n] for n in ss]):8.0f}")

# K2a (key-tile stationary dK/dV): one CTA's per-iteration timeline
buf = np.zeros((6, 512), dtype=np.int64)
fn = rt.lib().af_debug_bwd2a_trace
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p]
assert fn(buf.ctypes.data) == 0
names = ["mma: p_ready passed", "mma: ds_ready passed", "rows0: s_full passed",
         "rows0: P published", "rows0: dp_full passed", "rows0: dS published"]
nk = int((buf[2] > 0).sum())
ss = range(8, max(9, nk - 8))
base = buf[2]
print(f"K2a iterations traced {nk}; period (rows0 s_full to s_full): "
      f"{np.mean([buf[2, n + 1] - buf[2, n] for n in ss]):.0f} clk")
order = sorted(range(6), key=lambda e: np.mean([buf[e, n] - base[n] for n in ss]))
for e in order:
    print(f"  {names[e]:28s} {np.mean([buf[e, n] - base[n] for n in ss]):8.0f}")
