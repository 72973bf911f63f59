"""Developer probe (AF_TRACE build): per-role timeline of one backward CTA at cfg2 size."""
import ctypes, math, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
from paper_2502_15349_b200 import runtime as rt
from probe_bwd import desc
L = rt.lib()
B, H, Hk, S, D = 8, 32, 8, 8192, 128
dev = "cuda"
q = (torch.rand(B, H, S, D, device=dev) * 2 - 1).bfloat16()
k = (torch.rand(B, Hk, S, D, device=dev) * 2 - 1).bfloat16()
v = (torch.rand(B, Hk, S, D, device=dev) * 2 - 1).bfloat16()
do = (torch.rand(B, H, S, D, device=dev) * 2 - 1).bfloat16()
o = torch.empty_like(q); lse = torch.empty(B, H, S, device=dev)
d = desc(q, k, v, o, 1, 0, 0, 0, None)
assert L.af_parallel_fwd(d, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), None) == 0
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
n = L.af_parallel_bwd_workspace(d); ws = torch.empty(n, dtype=torch.uint8, device=dev)
for _ in range(2):
    assert L.af_parallel_bwd(d, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(),
                             dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), n, None) == 0
torch.cuda.synchronize()
buf = np.zeros((16, 512), dtype=np.int64)
fn = L.af_debug_trace_read; fn.restype = ctypes.c_int; fn.argtypes = [ctypes.c_void_p]
assert fn(buf.ctypes.data) == 0
names = ["mma:ds_ready(n)", "mma:p_ready(n)", "mma:dq_free(n-1)", "mma:full(n)", "wg:s_full", "wg:p_done",
         "wg:dp_full", "wg:ds_done", "dq:dq_full", "dq:tmem_freed", "tma:empty(n-2)"]
for it in (50, 51, 52, 120, 121):
    base = buf[0, it]
    print(f"iter {it}: period(ds_ready) {buf[0,it+1]-buf[0,it]} cycles")
    for e, nm in enumerate(names):
        print(f"   {nm:18s} {buf[e, it] - base:8d}")
per = np.diff(buf[0, 10:250])
print("median period", np.median(per), "mean", per.mean())
