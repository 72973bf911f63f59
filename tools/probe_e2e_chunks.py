"""Developer probe: the end-to-end (host-buffer) step of a config through HostPipeline at several
chunk counts — the PCIe-bound e2e leg's fill / drain shrinks with smaller chunks while the kernels
per chunk get smaller.  Usage: python tools/probe_e2e_chunks.py cfg2"""
import sys, json, torch
sys.path.insert(0, ".")
import bench
from paper_2502_15349_b200.pipeline import HostPipeline
key = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
spec = bench.build_spec(key)
w = bench.WORKLOADS[key]
dev = torch.device("cuda")
arrays, dout = bench.device_inputs(spec, dev, 0)
host = {k: v.cpu().pin_memory() for k, v in arrays.items()}
hdo = dout.cpu().pin_memory() if w.backward else None
wk = bench.work(spec)
flops = wk["fwd_flops"] + (wk["bwd_flops"] if w.backward else 0)
for mc, ov in ((16, True), (16, False), (8, True), (8, False), (16, True), (16, False)):
    pipe = HostPipeline(spec, device=dev, max_chunks=mc, overlap_calls=ov)
    out = pipe(host, hdo); pipe(host, hdo, out=out); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): pipe(host, hdo, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"cfg": key, "max_chunks": mc, "overlap_calls": ov, "units": len(pipe.units), "ms": round(ms, 2), "tflops": round(flops / ms / 1e9, 1)}))
    del pipe, out
    torch.cuda.empty_cache()
