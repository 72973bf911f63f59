"""Developer probe: K1 forward vs a torch fp64 reference on a few shapes, plus a cfg2 timing."""
import math, sys, time
import torch
sys.path.insert(0, "/root/repo")
from paper_2502_15349_b200 import runtime as rt

L = rt.lib()

def ref(q, k, v, causal, window, family, act, slope, scale):
    B, H, S, D = q.shape
    Hk = k.shape[1]
    g = H // Hk
    kk = k.double().repeat_interleave(g, 1); vv = v.double().repeat_interleave(g, 1)
    s = torch.einsum("bhid,bhjd->bhij", q.double(), kk) * scale
    Sq, Sk = q.shape[2], k.shape[2]
    i = torch.arange(Sq, device=q.device)[:, None]; j = torch.arange(Sk, device=q.device)[None, :]
    keep = torch.ones(Sq, Sk, dtype=torch.bool, device=q.device)
    if causal: keep &= j <= i
    if window > 0: keep &= (i - j) < window
    if family == 0:
        s = s.masked_fill(~keep, -math.inf)
        m = s.amax(-1, keepdim=True)
        p = torch.where(m == -math.inf, torch.zeros_like(s), torch.exp(s - m))
        l = p.sum(-1, keepdim=True)
        o = torch.where(l == 0, torch.zeros_like(l), 1 / l) * (p @ vv)
        lse = torch.where(l == 0, torch.full_like(l, -math.inf), m + torch.log(l)).squeeze(-1)
        return o, lse
    z = s
    if slope is not None: z = z - slope.double()[None, :, None, None] * (i - j)
    if act == 1: z = torch.sigmoid(z)
    elif act == 2: z = torch.relu(z)
    z = z * keep
    return z @ vv, None

def run(B, H, Hk, Sq, Sk, D, causal=0, window=0, family=0, act=0, slope=None, time_it=False):
    dev = "cuda"
    torch.manual_seed(0)
    q = (torch.rand(B, H, Sq, D, device=dev) * 2 - 1).bfloat16()
    k = (torch.rand(B, Hk, Sk, D, device=dev) * 2 - 1).bfloat16()
    v = (torch.rand(B, Hk, Sk, D, device=dev) * 2 - 1).bfloat16()
    o = torch.empty(B, H, Sq, D, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(B, H, Sq, device=dev, dtype=torch.float32)
    d = rt.ParallelDesc()
    d.batch, d.heads_q, d.heads_kv, d.seq_q, d.seq_k, d.d_qk, d.d_v = B, H, Hk, Sq, Sk, D, D
    d.dtype = 0
    d.q_stride, d.k_stride, d.v_stride, d.o_stride = rt.strides4(q), rt.strides4(k), rt.strides4(v), rt.strides4(o)
    d.family, d.act, d.scale = family, act, 1 / math.sqrt(D)
    d.causal, d.diag_offset, d.window = causal, 0, window
    d.slope = slope.data_ptr() if slope is not None else None
    d.bias = 0.0
    st = L.af_parallel_fwd(d, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), None)
    torch.cuda.synchronize()
    if st != 0:
        print("status", st, L.af_last_error()); return
    if time_it:
        for _ in range(3): L.af_parallel_fwd(d, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 10
        for _ in range(n): L.af_parallel_fwd(d, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), None)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        P = Sq * (Sq + 1) / 2 if causal else Sq * Sk
        fl = 2 * B * H * P * (2 * D)
        print(f"TIME B{B} H{H} S{Sq} D{D} causal={causal}: {ms:.3f} ms  {fl/ms/1e9:.1f} TFLOPS")
        return
    ro, rl = ref(q, k, v, causal, window, family, act, slope, 1 / math.sqrt(D))
    err = (o.double() - ro).abs().max().item()
    nrm = ((o.double() - ro).norm() / ro.norm().clamp_min(1e-30)).item()
    msg = f"B{B} H{H}/{Hk} Sq{Sq} Sk{Sk} D{D} c{causal} w{window} fam{family} act{act}: O maxabs {err:.2e} rel {nrm:.2e}"
    if rl is not None:
        fin = torch.isfinite(rl)
        le = (lse.double()[fin] - rl[fin]).abs().max().item() if fin.any() else 0.0
        msg += f" LSE {le:.2e} inf-match {bool(((lse == -math.inf) == (rl == -math.inf)).all())}"
    print(msg, flush=True)

if __name__ == "__main__":
    run(1, 1, 1, 256, 256, 128)
    run(1, 1, 1, 256, 256, 128, causal=1)
    run(1, 2, 1, 512, 512, 64, causal=1)
    run(2, 4, 2, 300, 300, 128, causal=1)
    run(1, 2, 2, 200, 333, 128)
    run(1, 2, 2, 1024, 1024, 128, causal=1, window=300)
    sl = torch.tensor([0.01, 0.003], device="cuda")
    run(1, 2, 2, 512, 512, 128, causal=1, window=200, family=1, act=1, slope=sl)
    run(1, 2, 2, 512, 512, 64, family=1, act=2)
    run(8, 32, 8, 8192, 8192, 128, causal=1, time_it=True)
    run(8, 32, 8, 8192, 8192, 128, causal=0, time_it=True)
