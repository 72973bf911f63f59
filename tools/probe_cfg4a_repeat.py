"""Developer probe: repeat the cfg4a (MLA, B1 H128 S4096) forward + backward at full shape and
count bitwise mismatches against the first run (the MLA path has no atomics, so any difference
is a race).  Prints the heads whose dQ differ and the largest relative difference."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
spec = configs.cfg4a()
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
o0, l0 = af.parallel_forward(spec, arrays)
g0 = af.parallel_backward(spec, arrays, o0, l0, dout)
fo = fb = 0
for it in range(reps):
    o, l = af.parallel_forward(spec, arrays)
    if not (torch.equal(o, o0) and torch.equal(l, l0)):
        fo += 1
        print("fwd mismatch heads:", (o != o0).flatten(2).any(-1)[0].nonzero().flatten()[:16].tolist())
    g = af.parallel_backward(spec, arrays, o0, l0, dout)
    for n in ("q", "k"):
        if not torch.equal(g[n], g0[n]):
            fb += 1
            d = (g[n].float() - g0[n].float())
            rel = (d.flatten(2).norm(dim=-1) / g0[n].float().flatten(2).norm(dim=-1).clamp_min(1e-30))
            bad = (rel > 0).nonzero()[:16].tolist()
            print(f"it {it} bwd d{n} mismatch (b,h): {bad} max rel {rel.max().item():.3e}")
            if n == "q":
                rows = (g[n] != g0[n]).any(-1)[0]
                print("   rows:", rows.nonzero()[:16].tolist())
print(f"forward mismatches {fo}/{reps}, backward mismatches {fb}/{reps}")

# localise: reuse one workspace (reuse_buffers) and compare its regions after each call
# [lse2 | delta | P | dS' | key-side partials] (mla_bwd_capi.cu mat_layout)
if fb:
    cache = {}
    with af.api.reuse_buffers(cache):
        af.parallel_backward(spec, arrays, o0, l0, dout)
        ws = [t for k_, t in cache.items() if k_[0] == "bwd.ws"][0]
        ref = ws.clone()
        rows = 128 * 4096
        stats, scores = rows * 8, rows * 4096 * 2
        regions = {"stats": (0, stats), "P": (stats, stats + scores),
                   "dS": (stats + scores, stats + 2 * scores), "part": (stats + 2 * scores, ws.numel())}
        for it in range(6):
            g = af.parallel_backward(spec, arrays, o0, l0, dout)
            torch.cuda.synchronize()
            msg = []
            for name, (a, b_) in regions.items():
                diff = (ws[a:b_] != ref[a:b_])
                nd = int(diff.sum().item())
                if nd:
                    first = int(diff.nonzero()[0].item())
                    if name in ("P", "dS"):
                        dv = (ws[a:b_].view(torch.bfloat16).view(128, 128, 32, 64, 64) !=
                              ref[a:b_].view(torch.bfloat16).view(128, 128, 32, 64, 64))
                        blk = dv.any(dim=4).any(dim=2).nonzero()  # (bh, 32-row slab, 64-col block)
                        msg.append(f"{name}: {nd} bytes differ in {blk.shape[0]} (bh, 32-row, "
                                   f"64-col) blocks: {blk[:12].tolist()}")
                    else:
                        msg.append(f"{name}: {nd} bytes differ (first byte {first})")
            print(f"ws run {it}:", "; ".join(msg) or "identical",
                  "| dq equal to first:", torch.equal(g["q"], g0["q"]))
