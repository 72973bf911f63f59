"""Developer probe: every benchmark config at its full shape, forward (and backward) repeated and
compared bit for bit with the first run — a race shows up as run-to-run differences long before
it shows up against a tolerance.  The parallel backward runs in deterministic (split K2a/K2b)
mode here; the fused 5-GEMM backward reduces dQ through L2 in arrival order (not bitwise
reproducible by design) and is compared against the split result within 1e-2 normwise."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2502_15349_b200 as af  # noqa: E402
from paper_2502_15349_b200.spec import Pattern  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
keys = sys.argv[2].split(",") if len(sys.argv) > 2 else ["cfg2", "cfg3", "cfg4a", "cfg4b", "cfg5a",
                                                          "cfg5b"]
dev = torch.device("cuda")
for key in keys:
    spec = bench.build_spec(key)
    w = bench.WORKLOADS[key]
    arrays, dout = bench.device_inputs(spec, dev, 0)
    par = spec.pattern is Pattern.PARALLEL

    def run():
        if par:
            o, lse = af.parallel_forward(spec, arrays)
            g = af.parallel_backward(spec, arrays, o, lse, dout) if w.backward else {}
            return o, lse, g
        o = af.linear_forward(spec, arrays)
        return o, None, af.linear_backward(spec, arrays, dout)

    af.use_deterministic_backward(True)
    o0, l0, g0 = run()
    bad = []
    for it in range(reps):
        o, l, g = run()
        if not torch.equal(o, o0) or (l0 is not None and not torch.equal(l, l0)):
            bad.append(f"fwd@{it}")
        for n in g0:
            if not torch.equal(g[n], g0[n]):
                rel = ((g[n].float() - g0[n].float()).norm() / g0[n].float().norm()).item()
                bad.append(f"d{n}@{it}:{rel:.1e}")
    af.use_deterministic_backward(False)
    extra = ""
    if par and w.backward:
        o, l, g = run()
        rel = {n: ((g[n].float() - g0[n].float()).norm() / g0[n].float().norm()).item()
               for n in g0}
        extra = " | default-mode vs split: " + " ".join(f"d{n} {r:.1e}" for n, r in rel.items())
    print(f"{key}: {'bitwise repeatable' if not bad else 'MISMATCH ' + ' '.join(bad[:8])}{extra}",
          flush=True)
    del arrays, dout, o0, l0, g0
    torch.cuda.empty_cache()
