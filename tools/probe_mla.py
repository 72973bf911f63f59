"""Developer probe: K3 MLA prefill/decode vs the f64 oracle (sampled rows) + cfg4 timing."""
import sys, math
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from dataclasses import replace
import oracle
from oracle import parallel as OP
import paper_2502_15349_b200 as af
from paper_2502_15349_b200 import spec as S

def mla_spec(b, h, sq, sk, causal):
    sp = S.builtin("softmax", batch=b, heads=h, heads_kv=1, seq_q=sq, seq_k=sk, d_qk=576, d_v=512)
    sp = replace(sp, kv_shared=True)
    return S.with_causal_mask(sp) if causal else sp

def run(b, h, sq, sk, causal, rows=None, time_it=False):
    sp = mla_spec(b, h, sq, sk, causal)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.rand(b, h, sq, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(b, 1, sk, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
    arrays = {"q": q, "k": k}
    o, lse = af.parallel_forward(sp, arrays)
    torch.cuda.synchronize()
    if time_it:
        for _ in range(3): af.parallel_forward(sp, arrays)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); n = 10
        for _ in range(n): af.parallel_forward(sp, arrays)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        P = sq * (sq + 1) / 2 if causal else sq * sk
        fl = 2 * b * h * P * (576 + 512)
        byts = b * sk * 576 * 2 + b * h * sq * (576 + 512) * 2
        print(f"TIME MLA B{b} H{h} Sq{sq} Sk{sk} causal={causal}: {ms:.3f} ms {fl/ms/1e9:.0f} TFLOPS {byts/ms/1e6:.0f} GB/s", flush=True)
        return
    rows = np.arange(sq) if rows is None else np.asarray(rows)
    errs, lerrs = [], []
    for bb in range(b):
        for hh in range(min(h, 6)):
            sub = mla_spec(1, 1, sq, sk, causal)
            a = {"q": q[bb:bb+1, hh:hh+1].double().cpu().numpy(), "k": k[bb:bb+1].double().cpu().numpy()}
            wo, wl = OP.sampled_forward(sub, a, rows)
            errs.append(np.abs(o[bb, hh, rows].double().cpu().numpy() - wo[0, 0]).max() / max(1, np.abs(wo).max()))
            lerrs.append(np.abs(lse[bb, hh, rows].double().cpu().numpy() - wl[0, 0]).max())
    print(f"MLA B{b} H{h} Sq{sq} Sk{sk} causal={causal}: O maxrel {max(errs):.2e} LSE {max(lerrs):.2e}", flush=True)

if __name__ == "__main__":
    run(1, 4, 300, 300, True)
    run(1, 2, 256, 256, False)
    run(2, 128, 1, 5000, False)
    run(1, 128, 1, 64, False)
    run(1, 128, 4096, 4096, True, time_it=True)
    run(16, 128, 1, 32768, False, time_it=True)
