"""Developer probe: repeat the MLA forward / backward at one shape and count bitwise mismatches."""
import sys
from dataclasses import replace
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200 import spec as S  # noqa: E402

b, h, sq, sk = 1, 5, 512, 512
spec = S.with_causal_mask(replace(S.builtin("softmax", batch=b, heads=h, heads_kv=1, seq_q=sq,
                                            seq_k=sk, d_qk=576, d_v=512), kv_shared=True))
g = torch.Generator(device="cuda").manual_seed(3)
q = (torch.rand(b, h, sq, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
k = (torch.rand(b, 1, sk, 576, device="cuda", generator=g) * 2 - 1).bfloat16()
dout = (torch.rand(b, h, sq, 512, device="cuda", generator=g) * 2 - 1).bfloat16()
o0, l0 = af.parallel_forward(spec, {"q": q, "k": k})
g0 = af.parallel_backward(spec, {"q": q, "k": k}, o0, l0, dout)
fo = fb = 0
for it in range(30):
    o, l = af.parallel_forward(spec, {"q": q, "k": k})
    if not (torch.equal(o, o0) and torch.equal(l, l0)):
        fo += 1
        bad = (o != o0).any(-1)[0]
        print("fwd mismatch rows (head, row):", bad.nonzero()[:8].tolist())
    gg = af.parallel_backward(spec, {"q": q, "k": k}, o0, l0, dout)
    if not (torch.equal(gg["q"], g0["q"]) and torch.equal(gg["k"], g0["k"])):
        fb += 1
        bad = (gg["q"] != g0["q"]).any(-1)[0]
        print("bwd dq mismatch rows:", bad.nonzero()[:8].tolist(), "dk rows",
              (gg["k"] != g0["k"]).any(-1)[0, 0].nonzero()[:8].flatten().tolist())
print(f"forward mismatches {fo}/30, backward mismatches {fb}/30")
