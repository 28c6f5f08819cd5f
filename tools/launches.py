"""Summarise an ncu --csv launch list (gpu__time_duration.sum): mean us per kernel name."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
acc = collections.OrderedDict()
for r in rows[1:]:
    k = r[ki].split("(")[0]
    acc.setdefault(k, []).append(float(r[vi].replace(",", "")) / 1000)
tot = 0
for k, v in acc.items():
    m = sum(v) / len(v)
    tot += m
    print(f"{k:45s} {m:9.1f} us  x{len(v)}")
print(f"{'sum of means':45s} {tot:9.1f} us")
