"""Stall reasons aggregated per SASS opcode for one kernel (ncu source page)."""
import csv, io, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si = hdr.index("Source")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.defaultdict(lambda: collections.Counter())
seen = set()
for r in rows[2:]:
    if len(r) <= sc[-1] or not r[sc[0]].isdigit() or r[0] in seen:
        continue
    seen.add(r[0])
    src = r[si].strip()
    op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
    for i in sc:
        agg[op][hdr[i][6:]] += int(r[i])
tot = sum(sum(c.values()) for c in agg.values())
for op, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:12]:
    s = sum(c.values())
    top = ", ".join(f"{k}={100*v/tot:.1f}" for k, v in c.most_common(5))
    print(f"{op:8s} {100*s/tot:5.1f}%  {top}")
