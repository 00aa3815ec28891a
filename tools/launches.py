"""Mean device time per kernel from an ncu --metrics gpu__time_duration.sum CSV."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
d = defaultdict(list)
for r in rows[1:]:
    if mi is not None and r[mi] != "gpu__time_duration.sum":
        continue
    try:
        d[r[ki][:70]].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
for k, v in d.items():
    print(f"{len(v):4d} x {sum(v) / len(v) / 1000:9.2f} us  {k}")
