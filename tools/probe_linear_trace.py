import ctypes, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import paper_2502_15349_b200 as af
from paper_2502_15349_b200 import runtime as rt, spec as S
name, dk = sys.argv[1], int(sys.argv[2])
b, h = 4, (16 if dk == 256 else 32)
sp = S.builtin(name, batch=b, heads=h, seq=8192, d_qk=dk, d_v=dk)
d = {"q": torch.rand(b, h, 8192, dk, device="cuda").bfloat16(), "k": torch.rand(b, h, 8192, dk, device="cuda").bfloat16(),
     "v": torch.rand(b, h, 8192, dk, device="cuda").bfloat16()}
for e in sp.extra_inputs:
    shp = e.resolve_shape(sp.dims)
    d[e.name] = (0.5 + 0.4 * torch.rand(*shp, device="cuda")) if e.fill == "unit" else torch.full(shp, 0.99, device="cuda")
for _ in range(2): af.linear_forward(sp, d)
torch.cuda.synchronize()
buf = np.zeros((16, 128), dtype=np.int64)
fn = rt.lib().af_debug_lin_trace_read; fn.restype = ctypes.c_int; fn.argtypes = [ctypes.c_void_p]
assert fn(buf.ctypes.data) == 0
names = ["mma:full", "mma:hb_ready(n-1)", "mma:p_ready", "mma:vw&h_scaled", "wg:(a) done", "wg:(b) vw done",
         "wg:(d) scaled", "wg:s_full", "wg:(c) P done", "wg:oi&qh", "wg:(e) done", "wg:h_full", "wg:(f) hb done", "wg:full passed", "wg:scan ready"]
for it in (10, 11, 40):
    base = buf[0, it]
    print(f"chunk {it}: period {buf[0, it+1] - base}")
    for e, nm in enumerate(names):
        print(f"   {nm:20s} {buf[e, it] - base:8d}")
