"""Developer probe: for the (bh, 32-row slab, 64-col block) tiles of the materialised MLA scores
(P) that differ between two backward runs, compare each run with P recomputed in fp32 from Q, K
and the forward LSE — and with P recomputed from the query rows of neighbouring tiles (a stale
TMEM buffer from tile n +- 1 / n +- 2 would match one of those)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import configs  # noqa: E402

spec = configs.cfg4a()
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
o0, l0 = af.parallel_forward(spec, arrays)
q, k = arrays["q"], arrays["k"]
scale = spec.scale if hasattr(spec, "scale") else 576 ** -0.5
rows = 128 * 4096
stats, scores = rows * 8, rows * 4096 * 2
cache = {}
with af.api.reuse_buffers(cache):
    af.parallel_backward(spec, arrays, o0, l0, dout)
    ws = [t for k_, t in cache.items() if k_[0] == "bwd.ws"][0]
    ref = ws.clone()
    lse2 = ws[:rows * 4].view(torch.float32).view(128, 4096)
    for it in range(3):
        af.parallel_backward(spec, arrays, o0, l0, dout)
        torch.cuda.synchronize()
        P = ws[stats:stats + scores].view(torch.bfloat16).view(128, 4096, 4096)
        R = ref[stats:stats + scores].view(torch.bfloat16).view(128, 4096, 4096)
        blk = (P.view(128, 128, 32, 64, 64) != R.view(128, 128, 32, 64, 64)).any(4).any(2).nonzero()
        print(f"run {it}: {blk.shape[0]} differing blocks")
        for bh, sl, cb in blk[:6].tolist():
            r0, c0 = sl * 32, cb * 64
            kk = k[0, 0, c0:c0 + 64].float()

            def p_from(rr):
                s = q[0, bh, rr:rr + 32].float() @ kk.T
                return torch.exp2(s * (scale * 1.4426950408889634) - lse2[bh, r0:r0 + 32, None])

            want = p_from(r0)
            got, old = P[bh, r0:r0 + 32, c0:c0 + 64].float(), R[bh, r0:r0 + 32, c0:c0 + 64].float()
            bad_rows = (got != old).any(1).nonzero().flatten().tolist()
            line = (f"  bh {bh} rows {r0}+{bad_rows[:4]}..({len(bad_rows)}) cols {c0}: "
                    f"|new-true| {(got - want).abs().max().item():.3e} "
                    f"|old-true| {(old - want).abs().max().item():.3e}")
            for dr in (-256, -128, 128, 256):
                if 0 <= r0 + dr < 4096:
                    alt = p_from(r0 + dr)
                    line += f" | new vs rows{dr:+d} {(got - alt).abs().max().item():.2e}"
            print(line)
            nz = (got != old)
            print("     differing entries:", int(nz.sum()), "of 2048; sample new/old/true:",
                  [(round(a, 4), round(b, 4), round(c, 4)) for a, b, c in
                   zip(got[nz][:3].tolist(), old[nz][:3].tolist(), want[nz][:3].tolist())])
