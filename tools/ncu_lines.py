"""Warp-stall samples per CUDA source line for one kernel (ncu source page, cuda+sass view).
usage: python tools/ncu_lines.py rep.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, res = "?", []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 6 and r[0].isdigit() and r[4].isdigit():
        res.append((int(r[4]), fname, int(r[0]), r[1].strip()[:90], r[7]))
tot = sum(x[0] for x in res) or 1
for s, f, ln, src, ie in sorted(res, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{ln:<5d} inst={ie:>10s}  {src}")
