"""Developer probe: K4/K5 linear template vs the f64 oracle, plus cfg5 timing."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import oracle
from oracle import recurrent as OR
import paper_2502_15349_b200 as af
from paper_2502_15349_b200 import spec as S

def dev(a):
    return {k: torch.tensor(v, device="cuda").to(torch.bfloat16 if k in "qkv" else torch.float32) for k, v in a.items()}

def rounded(a):
    out = dict(a)
    for k in "qkv":
        out[k] = torch.tensor(a[k]).to(torch.bfloat16).double().numpy()
    return out

def nw(g, w):
    return float(np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-30))

def check(name, b, h, s, dk, dv):
    sp = S.builtin(name, batch=b, heads=h, seq=s, d_qk=dk, d_v=dv)
    a = oracle.generate(sp, 5)
    d = dev(a)
    o = af.linear_forward(sp, d)
    ra = rounded(a)
    want = OR.chunk_forward(sp, ra, 64)
    msg = f"{name} B{b} H{h} S{s} {dk}/{dv}: fwd nw {nw(o.double().cpu().numpy(), want):.2e}"
    dout = np.random.default_rng(1).uniform(-1, 1, want.shape)
    dt = torch.tensor(dout, device="cuda").to(torch.bfloat16)
    g = af.linear_backward(sp, d, dt)
    gw = OR.chunk_vjp(sp, ra, dt.double().cpu().numpy(), chunk=64)
    for k in gw:
        msg += f" d{k} {nw(g[k].double().cpu().numpy().reshape(gw[k].shape), gw[k]):.2e}"
    print(msg, flush=True)

def timeit(name, b, h, s, dk, dv):
    sp = S.builtin(name, batch=b, heads=h, seq=s, d_qk=dk, d_v=dv)
    a = {k: torch.tensor(v, device="cuda") for k, v in oracle.generate(S.builtin(name, batch=1, heads=1, seq=8, d_qk=4, d_v=4), 0).items()}
    g = torch.Generator(device="cuda").manual_seed(0)
    d = {"q": (torch.rand(b, h, s, dk, device="cuda", generator=g) * 2 - 1).bfloat16(),
         "k": (torch.rand(b, h, s, dk, device="cuda", generator=g) * 2 - 1).bfloat16(),
         "v": (torch.rand(b, h, s, dv, device="cuda", generator=g) * 2 - 1).bfloat16()}
    for e in sp.extra_inputs:
        shp = e.resolve_shape(sp.dims)
        if e.fill == "unit":
            d[e.name] = 0.5 + 0.45 * (torch.rand(*shp, device="cuda") * 2 - 1)
        else:
            gm = torch.tensor(e.fill_params["gamma"], device="cuda", dtype=torch.float32)
            d[e.name] = gm.view(1, -1, 1, 1).expand(*shp).contiguous()
    dout = torch.rand(b, h, s, dv, device="cuda").bfloat16()
    for _ in range(3):
        af.linear_forward(sp, d); af.linear_backward(sp, d, dout)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    n = 5
    e0.record()
    for _ in range(n): af.linear_forward(sp, d)
    e1.record()
    for _ in range(n): af.linear_backward(sp, d, dout)
    e2.record(); torch.cuda.synchronize()
    f, bw = e0.elapsed_time(e1) / n, e1.elapsed_time(e2) / n
    fb = b * h * s * (2 * dk + 2 * dv) * 2  # q,k,v,o bf16
    print(f"TIME {name} B{b} H{h} S{s} {dk}/{dv}: fwd {f:.3f} ms ({fb/f/1e6:.0f} GB/s), bwd {bw:.3f} ms", flush=True)

if __name__ == "__main__":
    check("retention-recurrent", 1, 2, 384, 128, 128)
    check("mamba2-ssm", 1, 2, 300, 128, 128)
    check("gated-retention", 1, 2, 256, 256, 256)
    check("retention-recurrent", 2, 1, 512, 256, 256)
    check("mamba2-ssm", 1, 1, 1000, 128, 256)
    timeit("retention-recurrent", 4, 16, 8192, 256, 256)
    timeit("mamba2-ssm", 4, 32, 8192, 128, 128)
