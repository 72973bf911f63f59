"""Library yardstick (not the product): torch SDPA (cuDNN / flash backends) fwd+bwd at cfg2/cfg3
shapes on this B200, timed with CUDA events — tells how far our K1/K2 sit from NVIDIA's own
sm_100 kernels on the same box.  Prints one JSON line per backend."""
import json
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

B, HQ, HKV, S, D = 8, 32, 8, 8192, 128
dev = "cuda"
q = torch.randn(B, HQ, S, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
k = torch.randn(B, HKV, S, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
v = torch.randn(B, HKV, S, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
do = torch.randn(B, HQ, S, D, device=dev, dtype=torch.bfloat16)
pairs = B * HQ * S * (S + 1) / 2
fwd_fl, bwd_fl = 4 * D * pairs, 10 * D * pairs
for name, be in [("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)]:
    try:
        with sdpa_kernel([be]):
            def step():
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
                return o
            for _ in range(3):
                o = step(); o.backward(do)
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            fm = bm = 0.0
            n = 5
            for _ in range(n):
                e[0].record(); o = step(); e[1].record(); o.backward(do); e[2].record()
                torch.cuda.synchronize()
                fm += e[0].elapsed_time(e[1]); bm += e[1].elapsed_time(e[2])
            fm /= n; bm /= n
            print(json.dumps({"backend": name, "fwd_ms": fm, "bwd_ms": bm,
                              "fwd_tflops": fwd_fl / fm / 1e9, "bwd_tflops": bwd_fl / bm / 1e9}))
    except Exception as ex:  # noqa: BLE001
        print(json.dumps({"backend": name, "error": str(ex)[:200]}))
