"""profiles/traffic_<workload>.json from an ncu --csv log of
dram__bytes_read.sum / dram__bytes_write.sum / gpu__time_duration.sum
(cold-cache, serialised launches of bench.py):
python tools/traffic_json.py gpurun_out/traffic.csv profiles/traffic_c2.json "<source>" """
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
acc = defaultdict(lambda: defaultdict(list))
for r in rows[1:]:
    try:
        acc[r[ki].split("(")[0]][r[mi]].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
out = {"source": sys.argv[3] if len(sys.argv) > 3 else sys.argv[1], "kernels": {}}
total = 0.0
for k, m in acc.items():
    rd = sum(m["dram__bytes_read.sum"]) / len(m["dram__bytes_read.sum"])
    wr = sum(m["dram__bytes_write.sum"]) / len(m["dram__bytes_write.sum"])
    us = sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"]) / 1e3
    out["kernels"][k] = {"dram_read": rd, "dram_write": wr,
                         "launches": len(m["dram__bytes_read.sum"]), "us": us}
    total += rd + wr
out["bytes_per_step"] = total
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
