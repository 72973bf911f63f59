"""Developer probe: K2 backward vs torch fp64 autograd, plus cfg2 timing."""
import math, sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2502_15349_b200 import runtime as rt
from probe_fwd import ref
L = rt.lib()

def desc(q, k, v, o, causal, window, family, act, slope):
    B, H, Sq, D = q.shape
    d = rt.ParallelDesc()
    d.batch, d.heads_q, d.heads_kv, d.seq_q, d.seq_k, d.d_qk, d.d_v = B, H, k.shape[1], Sq, k.shape[2], D, v.shape[3]
    d.dtype = 0
    d.q_stride, d.k_stride, d.v_stride, d.o_stride = rt.strides4(q), rt.strides4(k), rt.strides4(v), rt.strides4(o)
    d.family, d.act, d.scale = family, act, 1 / math.sqrt(D)
    d.causal, d.diag_offset, d.window = causal, 0, window
    d.slope = slope.data_ptr() if slope is not None else None
    d.bias = 0.0
    return d

def run(B, H, Hk, Sq, Sk, D, causal=0, window=0, family=0, act=0, slope=None, time_it=False):
    dev = "cuda"
    torch.manual_seed(1)
    q = (torch.rand(B, H, Sq, D, device=dev) * 2 - 1).bfloat16()
    k = (torch.rand(B, Hk, Sk, D, device=dev) * 2 - 1).bfloat16()
    v = (torch.rand(B, Hk, Sk, D, device=dev) * 2 - 1).bfloat16()
    do = (torch.rand(B, H, Sq, D, device=dev) * 2 - 1).bfloat16()
    o = torch.empty(B, H, Sq, D, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(B, H, Sq, device=dev, dtype=torch.float32)
    d = desc(q, k, v, o, causal, window, family, act, slope)
    st = L.af_parallel_fwd(d, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), None)
    assert st == 0, L.af_last_error()
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws_n = L.af_parallel_bwd_workspace(d)
    ws = torch.empty(ws_n, dtype=torch.uint8, device=dev)
    call = lambda: L.af_parallel_bwd(d, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(),
                            dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws_n, None)
    st = call(); torch.cuda.synchronize()
    if st != 0:
        print("status", st, L.af_last_error()); return
    if time_it:
        for _ in range(2): call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); n = 5
        for _ in range(n): call()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        P = Sq * (Sq + 1) / 2 if causal else Sq * Sk
        fl = 2 * B * H * P * (3 * D + 2 * D)
        print(f"BWD TIME B{B} H{H} S{Sq} D{D} causal={causal}: {ms:.3f} ms  {fl/ms/1e9:.1f} TFLOPS", flush=True)
        return
    qd, kd, vd = (x.double().requires_grad_() for x in (q, k, v))
    ro, _ = ref(qd, kd, vd, causal, window, family, act, slope, 1 / math.sqrt(D))
    ro.backward(do.double())
    msg = f"B{B} H{H}/{Hk} Sq{Sq} Sk{Sk} D{D} c{causal} w{window} fam{family} act{act}:"
    for name, got, want in (("dq", dq, qd.grad), ("dk", dk, kd.grad), ("dv", dv, vd.grad)):
        rel = ((got.double() - want).norm() / want.norm().clamp_min(1e-30)).item()
        mx = (got.double() - want).abs().max().item()
        msg += f" {name} rel {rel:.2e} max {mx:.2e};"
    print(msg, flush=True)

if __name__ == "__main__":
    run(1, 1, 1, 128, 128, 128)
    run(1, 1, 1, 256, 256, 128, causal=1)
    run(1, 2, 1, 512, 512, 64, causal=1)
    run(2, 4, 2, 300, 300, 128, causal=1)
    run(1, 2, 2, 200, 333, 128)
    run(1, 2, 2, 1024, 1024, 128, causal=1, window=300)
    sl = torch.tensor([0.01, 0.003], device="cuda")
    run(1, 2, 2, 512, 512, 128, causal=1, window=200, family=1, act=1, slope=sl)
    run(1, 2, 2, 512, 512, 64, family=1, act=2)
    run(8, 32, 8, 8192, 8192, 128, causal=1, time_it=True)
