"""Summarise an ncu report's SASS page: top instructions by warp-stall samples + stall mix."""
import csv, subprocess, sys, collections

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
tot = collections.Counter()
op = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    st = {h: int(r[idx[h]] or 0) for h in stalls}
    for h, v in st.items():
        tot[h] += v
    opc = r[idx["Source"]].split()[0] if r[idx["Source"]].split() else "?"
    if opc.startswith("@"):
        opc = r[idx["Source"]].split()[1]
    op[opc.split(".")[0]] += s
    data.append((s, r[idx["Address"]], r[idx["Source"]].strip(), max(st, key=st.get)))
T = sum(tot.values()) or 1
print("stall mix:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in tot.most_common(10)))
print("by opcode:", ", ".join(f"{k} {100*v/T:.1f}%" for k, v in op.most_common(14)))
for s, a, src, top in sorted(data, reverse=True)[:n]:
    print(f"{100*s/T:5.1f}%  {top[6:]:14s} {src[:90]}")
