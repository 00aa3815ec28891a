"""Mean of every metric per kernel from an `ncu --metrics ... --csv` log."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"),
                  h.index("Metric Value"), h.index("Metric Unit"))
d = defaultdict(lambda: defaultdict(list))
for r in rows[1:]:
    try:
        d[r[ki][:60]][(r[mi], r[ui])].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
for k, m in d.items():
    n = max(len(v) for v in m.values())
    print(f"{n:3d} x {k}")
    for (name, unit), v in sorted(m.items()):
        print(f"      {name:40s} {sum(v) / len(v):14.3f} {unit}")
