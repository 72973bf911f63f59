"""Developer probe: HostPipeline e2e timing vs chunk count, and the box's raw PCIe rates
(H2D alone, D2H alone, both at once) for the same byte counts."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_2502_15349_b200.pipeline import HostPipeline


def timed(fn, n=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for key in sys.argv[1:] or ["cfg2"]:
    w = bench.WORKLOADS[key]
    spec = bench.build_spec(key)
    arrays, dout = bench.device_inputs(spec, torch.device("cuda"), 0)
    host = {k: v.cpu().pin_memory() for k, v in arrays.items()}
    hdo = dout.cpu().pin_memory() if w.backward else None
    if hdo is not None:
        host_all = dict(host, dout=hdo)
    else:
        host_all = host
    tot = sum(t.numel() * t.element_size() for t in host_all.values())
    dev = {k: torch.empty_like(v, device="cuda") for k, v in host_all.items()}
    back = {k: torch.empty_like(v).pin_memory() for k, v in host_all.items()}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        for k in host_all:
            dev[k].copy_(host_all[k], non_blocking=True)

    def d2h():
        for k in host_all:
            back[k].copy_(dev[k], non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            h2d()
        with torch.cuda.stream(s2):
            d2h()
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    for name, fn in (("H2D", h2d), ("D2H", d2h), ("H2D+D2H", both)):
        ms = timed(fn)
        print(f"{key}: {name} {tot / 1e6:.0f} MB each way: {ms:.1f} ms "
              f"({tot / ms / 1e6:.1f} GB/s per direction)", flush=True)
    import time
    for chunks in (8, 16, 32):
        pipe = HostPipeline(spec, max_chunks=chunks)
        out = pipe(host, hdo)
        ms = timed(lambda: pipe(host, hdo, out=out))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pipe(host, hdo, out=out)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{key}: pipeline {len(pipe.units)} chunks: {ms:.1f} ms (enqueue {1e3 * (t1 - t0):.1f} "
              f"ms, wall {1e3 * (t2 - t0):.1f} ms)", flush=True)
    # the same pipeline with the kernels only (inputs already on device): the compute share
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        pipe(host, hdo, out=out)
        torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"],
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    for e in evs[:80]:
        print(f"  {e.name[:40]:40s} start {(e.time_range.start - t0) / 1e3:8.2f} ms  dur "
              f"{(e.time_range.end - e.time_range.start) / 1e3:7.2f} ms")
