"""Developer probe: K3b MLA backward vs the f64 oracle (small) + cfg4a fwd/bwd timing."""
import sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from oracle import parallel as OP
import paper_2502_15349_b200 as af
from paper_2502_15349_b200 import configs as C

def check(b, h, s, causal=True):
    sp = C.mla(b, h, s, s, causal)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.rand(b, h, s, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(b, 1, s, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
    o, lse = af.parallel_forward(sp, {"q": q, "k": k})
    do = (torch.rand(b, h, s, 512, device="cuda", generator=g) * 2 - 1).bfloat16()
    gr = af.parallel_backward(sp, {"q": q, "k": k}, o, lse, do)
    torch.cuda.synchronize()
    w = OP.parallel_vjp(sp, {"q": q.double().cpu().numpy(), "k": k.double().cpu().numpy()}, do.double().cpu().numpy())
    for n in ("q", "k"):
        gg = gr[n].double().cpu().numpy()
        print(f"MLA bwd B{b} H{h} S{s} causal={causal} d{n}: normwise {np.linalg.norm(gg-w[n])/np.linalg.norm(w[n]):.2e} maxabs {np.abs(gg-w[n]).max():.2e} |ref| {np.abs(w[n]).max():.2e}", flush=True)

def timeit():
    sp = C.cfg4a()
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.rand(1, 128, 4096, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(1, 1, 4096, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
    do = (torch.rand(1, 128, 4096, 512, device="cuda", generator=g) * 2 - 1).bfloat16()
    o, lse = af.parallel_forward(sp, {"q": q, "k": k})
    for _ in range(3): af.parallel_backward(sp, {"q": q, "k": k}, o, lse, do)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): af.parallel_backward(sp, {"q": q, "k": k}, o, lse, do)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"TIME MLA bwd cfg4a: {ms:.3f} ms = {5.911e12/ms/1e9:.0f} TFLOPS", flush=True)

if __name__ == "__main__":
    check(1, 2, 256)
    check(1, 3, 200, causal=False)
    check(1, 4, 300)
    timeit()
