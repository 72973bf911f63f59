"""Developer probe: HostPipeline e2e timing breakdown (CPU enqueue time vs device time)."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_2502_15349_b200.pipeline import HostPipeline

for key in sys.argv[1:] or ["cfg5b", "cfg2"]:
    w = bench.WORKLOADS[key]
    spec = bench.build_spec(key)
    arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
    host = {k: v.cpu().pin_memory() for k, v in arrays.items()}
    hdo = dout.cpu().pin_memory() if w.backward else None
    pipe = HostPipeline(spec)
    out = pipe(host, hdo)
    torch.cuda.synchronize()
    for it in range(3):
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe(host, hdo, out=out)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{key}: enqueue {1e3*(t1-t0):.1f} ms, device {e0.elapsed_time(e1):.1f} ms, wall {1e3*(t2-t0):.1f} ms", flush=True)
    # plain copies for reference
    tot = sum(t.numel() * t.element_size() for t in host.values())
    dev = {k: torch.empty_like(v, device="cuda") for k, v in host.items()}
    e0.record()
    for k in host: dev[k].copy_(host[k], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(f"{key}: plain H2D {tot/1e6:.0f} MB in {e0.elapsed_time(e1):.1f} ms", flush=True)
