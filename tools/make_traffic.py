"""profiles/roofline_traffic.json from the round's ncu summaries: DRAM read + write bytes per
launch of every kernel of one config step, summed into the forward and backward shares the bench's
roofline.traffic reports.  Usage: python tools/make_traffic.py TAG (reads
profiles/ncu_summary_TAG_<cfg>.json)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1]
FWD = ("parallel_fwd_kernel", "mla_fwd_kernel", "mla_combine_kernel", "parallel_fwd_f32")
out = {"source": f"ncu --set full captures of one step per config (tools/run_step_once.py), "
                 f"profiles/ncu_summary_{tag}_<cfg>.json", "tag": tag}
for cfg in ("cfg1", "cfg2", "cfg3", "cfg4a", "cfg4b", "cfg5a", "cfg5b"):
    p = ROOT / "profiles" / f"ncu_summary_{tag}_{cfg}.json"
    if not p.exists():
        continue
    doc = json.loads(p.read_text())
    out["head"] = doc.get("head")
    recs = [r for k, v in doc.items() if k.endswith(".ncu-rep") for r in v]
    per, fwd, bwd = {}, 0.0, 0.0
    linear = cfg.startswith("cfg5")
    seen_chunk = 0
    # the library's kernels only (the captures filter on the demangled "af::" name; the summary
    # keeps ncu's function base name)
    recs = [r for r in recs if "at::" not in r["kernel"] and "elementwise" not in r["kernel"]]
    for i, r in enumerate(recs):
        name = r["kernel"].split("(")[0].replace("void ", "").replace("af::", "")
        name = name.split("<")[0].split("::")[-1] + ("<" + name.split("<", 1)[1] if "<" in name
                                                        and "unnamed>" not in name else "")
        nbytes = r.get("dram_read_bytes", 0.0) + r.get("dram_write_bytes", 0.0)
        per[f"{name}#{i}"] = nbytes
        if linear:  # launch order: scan, forward chunk kernel | backward passes
            chunk = "linear_chunk" in name or "linear_wide" in name
            is_fwd = seen_chunk == 0 and ("decay_scan" in name or chunk)
            if chunk:
                seen_chunk += 1
        else:
            is_fwd = name.startswith(FWD)
        if is_fwd:
            fwd += nbytes
        else:
            bwd += nbytes
    out[cfg] = {"per_kernel_dram_bytes": per, "fwd_dram_bytes_per_launch": fwd}
    if bwd:
        out[cfg]["bwd_dram_bytes_per_launch"] = bwd
(ROOT / "profiles" / "roofline_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps({k: v for k, v in out.items() if k.startswith("cfg")}, indent=1)[:3000])
