"""Developer timeline of one K1 CTA (build with AF_EXTRA_NVCC_FLAGS=-DAF_FWD_TRACE).

Prints per-iteration SM-clock deltas for the row warps (S wait -> TMEM load -> P published) and
the MMA warp (waits on P of tile 0 / tile 1), averaged over the steady-state iterations.
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import runtime as rt  # noqa: E402

spec = bench.build_spec("cfg2")
dev = torch.device("cuda", 0)
arrays, _ = bench.device_inputs(spec, dev, 0)
for _ in range(3):
    af.parallel_forward(spec, arrays)
torch.cuda.synchronize()
lib = rt.lib()
buf = (C.c_ulonglong * (9 * 64 * 6 + 1))()
assert lib.af_debug_fwd_trace(buf, len(buf)) == 0
t = np.array(buf[:9 * 64 * 6], dtype=np.int64).reshape(9, 64, 6)
rows, mma = t[:8], t[8]
ss = slice(8, 56)
names = ["S wait->ldtm", "ldtm->max", "max->P half 0 (split: ->P stored)", "->P half 1 stored", "->published"]
for w in (0, 4):
    d = np.diff(rows[w, ss, :], axis=1).mean(axis=0)
    print(f"tile{w // 4} warp0:", ", ".join(f"{n} {v:.0f}" for n, v in zip(names, d)))
    print(f"  published -> next S ready {np.mean(rows[w, 9:57, 0] - rows[w, ss, 5]):.0f}; "
          f"period {np.diff(rows[w, :, 0])[ss].mean():.0f}")
print(f"mma: v_full done -> p0 {np.mean(mma[ss, 1] - mma[ss, 0]):.0f}, "
      f"p0 -> p1 {np.mean(mma[ss, 2] - mma[ss, 1]):.0f}, "
      f"p1 -> next vfull {np.mean(mma[9:57, 0] - mma[ss, 2]):.0f}")
