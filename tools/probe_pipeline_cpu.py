"""Developer probe: where the host spends time enqueueing one HostPipeline call (cProfile)."""
import cProfile, pstats, sys
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_2502_15349_b200.pipeline import HostPipeline

key = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = bench.WORKLOADS[key]
spec = bench.build_spec(key)
arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
host = {k: v.cpu().pin_memory() for k, v in arrays.items()}
hdo = dout.cpu().pin_memory() if w.backward else None
pipe = HostPipeline(spec)
out = pipe(host, hdo)
pipe(host, hdo, out=out)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    pipe(host, hdo, out=out)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
