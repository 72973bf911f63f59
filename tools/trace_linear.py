"""Developer timeline of one linear-template CTA (build with AF_EXTRA_NVCC_FLAGS=-DAF_TRACE).

Prints SM-clock stamps of the chunk pipeline (relative to the row warps' scan_ready pass of the
chunk) averaged over steady-state chunks, for the forward kernel of cfg5a / cfg5b."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import runtime as rt  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg5b"
bwd = len(sys.argv) > 2 and sys.argv[2] == "bwd"  # trace the last chunk-kernel run of the VJP
spec = bench.build_spec(key)
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
for _ in range(3):
    if bwd:
        af.linear_backward(spec, arrays, dout)
    else:
        af.linear_forward(spec, arrays)
torch.cuda.synchronize()
buf = np.zeros((24, 128), dtype=np.int64)
fn = rt.lib().af_debug_lin_trace_read
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p]
assert fn(buf.ctypes.data) == 0
names = {15: "scan: scan_ready arrive", 14: "rows: scan_ready passed", 4: "rows: cp handed",
         13: "rows: vfull passed", 5: "rows: Vw written", 6: "rows: H scaled",
         7: "rows: s_full passed", 8: "rows: P written", 11: "rows: h_full+qh_full passed",
         12: "rows: bf16 H written", 0: "mma: Q/K full", 1: "mma: hb_ready+oi_empty",
         3: "mma: vw+h_scaled", 2: "mma: p_ready+vfull", 9: "out: oi_full passed",
         10: "out: O written", 16: "prod: scan_free passed", 17: "prod: raw landed",
         18: "rows: scan stored", 19: "rows: row factors done"}
if len(sys.argv) > 3 and sys.argv[3] == "wide":  # linear_wide_kernel event map
    names = {15: "prod: empty passed", 14: "rows: full passed", 0: "mma: full (S issued)",
             1: "mma: hb_ready (QH issued)", 3: "mma: pk+h_scaled (H upd)",
             2: "mma: o_scaled (OI)", 7: "rows: s_full passed", 8: "rows: P+Kw done",
             11: "rows: qh_full passed", 12: "rows: O scaled", 9: "out: oi_full passed",
             10: "out: O written", 16: "state: h_full passed", 17: "state: Hb + H*g done"}
ss = range(8, 56)
base = buf[14]
period = np.mean([buf[14, n + 1] - buf[14, n] for n in ss])
print(f"{key}: steady chunk period {period:.0f} clk")
order = sorted(names, key=lambda e: np.mean([buf[e, n] - base[n] for n in ss]))
for e in order:
    rel = np.mean([buf[e, n] - base[n] for n in ss])
    print(f"  {names[e]:28s} {rel:8.0f}")
