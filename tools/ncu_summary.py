"""Condense ncu reports into the JSON/markdown summaries committed under profiles/."""
import csv, io, json, subprocess, sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "tensor_pipe_active_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "mem_throughput_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "smem_dynamic_kb": "launch__shared_mem_per_block_dynamic",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
# gpu__time_duration is reported in ns, us (usecond), ms (msecond) or s depending on magnitude
TO_MS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")}
        for k, m in KEYS.items():
            if m not in d:
                continue
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:  # "no data" for metrics a short kernel did not report
                continue
            if k.endswith("_bytes"):
                v *= SCALE.get(u[m], 1.0)
            elif k == "duration_ms":
                if u[m] not in TO_MS:
                    raise ValueError(f"unknown duration unit {u[m]!r}")
                v *= TO_MS[u[m]]
            rec[k] = v
        res.append(rec)
    return res


def launches(csv_path):
    lines = [ln for ln in open(csv_path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    tot = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        v *= TO_MS[unit]
        tot.setdefault(name, []).append(v)
    return {k: {"launches": len(v), "ms_total": sum(v), "ms_avg": sum(v) / len(v)}
            for k, v in tot.items()}


if __name__ == "__main__":
    import os
    from pathlib import Path
    head = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True,
                          text=True).stdout.strip()
    sha_file = Path(__file__).resolve().parents[1] / ".head_sha"  # written before a gpurun call
    if not head and sha_file.exists():  # (the GPU box's copy of the repo has no .git)
        head = sha_file.read_text().strip()
    head = os.environ.get("AF_HEAD", head)
    out = {"head": head}
    for rep in sys.argv[1:]:
        if rep.endswith(".csv"):
            out["launch_list"] = launches(rep)
        else:
            out[rep.split("/")[-1]] = summarize(rep)
    print(json.dumps(out, indent=1))
