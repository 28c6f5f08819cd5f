"""Top SASS lines of one kernel by warp-stall samples (ncu -i rep --page source --csv)."""
import csv, io, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si, ni, ei = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [(int(r[ni] or 0), int(r[ei] or 0), r[si].strip(), i) for i, r in enumerate(rows[2:]) if len(r) > ei and r[ni].isdigit()]
tot = sum(d[0] for d in data)
byop = collections.Counter()
exe = collections.Counter()
for s, e, src, _ in data:
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    byop[op] += s
    exe[op] += e
print(f"total samples {tot}")
for op, s in byop.most_common(15):
    print(f"  {op:10s} {100*s/tot:5.1f}%  executed {exe[op]}")
print("top lines:")
for s, e, src, i in sorted(data, reverse=True)[:top]:
    print(f"  {100*s/tot:5.1f}%  #{i:5d} exe {e:8d}  {src[:90]}")
