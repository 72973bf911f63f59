"""Developer probe (library built with AF_EXTRA_NVCC_FLAGS=-DAF_SCORES_TRACE): wait accounting of
the materialised-backward scores kernel at cfg4a — per CTA, the MMA thread's cycles waiting for
the operand boxes (k_ready), S^T / dP^T release (s_free / dp_free), ring data (full) and its
total; key-row warp 0's waits for statistics, S^T and dP^T — averaged over the traced CTAs."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import configs, runtime as rt  # noqa: E402

spec = configs.cfg4a()
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
o, lse = af.parallel_forward(spec, arrays)
af.parallel_backward(spec, arrays, o, lse, dout)
torch.cuda.synchronize()
L = rt.lib()
buf = np.zeros((256, 8), np.int64)
L.af_debug_scores_trace(ctypes.c_void_p(buf.ctypes.data), 1)
af.parallel_backward(spec, arrays, o, lse, dout)
torch.cuda.synchronize()
L.af_debug_scores_trace(ctypes.c_void_p(buf.ctypes.data), 0)
lead = buf[0::2]
names = ["mma: k_ready", "mma: s_free", "mma: full", "mma: dp_free", "mma: total",
         "row0: stat_full", "row0: s_full", "row0: dp_full"]
for i, nm in enumerate(names):
    src = lead if i <= 4 else buf
    v = src[:, i]
    v = v[v > 0] if i == 4 else v
    print(f"{nm:16s} mean {v.mean():12.0f} clk")
tot = lead[:, 4][lead[:, 4] > 0]
print("MMA-thread busy fraction (total - waits) / total:",
      float(((lead[:, 4] - lead[:, 0] - lead[:, 1] - lead[:, 2] - lead[:, 3])[lead[:, 4] > 0] / tot).mean()))
