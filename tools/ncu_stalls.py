"""Top warp-stall reasons per kernel from an ncu report (cycles per issued instruction)."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
ki = h.index("Kernel Name")
cols = [i for i, c in enumerate(h) if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for row in r[2:]:
    if pat in row[ki]:
        vals = sorted([(float(row[i].replace(",", "") or 0), h[i][len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                       for i in cols if row[i] not in ("", "n/a")], reverse=True)[:7]
        print(f"{row[ki][:30]:30s} " + "  ".join(f"{n}={v:.2f}" for v, n in vals))
