"""profiles/traffic.json from an ncu --set full report of the C3 kernels: DRAM bytes (read + write)
per launch of each stage (one launch each).  usage: python tools/traffic_from_ncu.py rep.ncu-rep tag"""
import csv
import io
import json
import subprocess
import sys

NAMES = [("k1c_fwd", "K1"), ("k2c_fwd", "K2"), ("k3_ring", "K3"), ("k4c_dct<512, 0>", "K4"),
         ("k5_ring", "K5"), ("k5t_ring", "K5T"), ("k4c_dct<512, 1>", "K4T"), ("k3t_ring", "K3T"),
         ("k2t_strip", "K2Ta"), ("k2t_sum", "K2Ta"), ("k2c_adjf", "K2Tb"), ("k2c_adj", "K2Tb"),
         ("k1c_adj", "K1T")]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
ki, r_i, w_i = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {}
for r in rows[2:]:
    for pat, st in NAMES:
        if pat in r[ki] and st not in res:
            res[st] = (float(r[r_i]) * scale.get(units[r_i], 1) + float(r[w_i]) * scale.get(units[w_i], 1))
            break
res["K2T"] = res.get("K2Ta", 0.0) + res.get("K2Tb", 0.0)
json.dump({"C3": res, "source": f"{sys.argv[2]} (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum "
           "per launch; K2Ta = k2t_strip, K2Tb = k2c_adj, K2T = their sum)"},
          open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(res, indent=1))
