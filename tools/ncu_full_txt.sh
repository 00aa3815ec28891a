# text summary of a full ncu capture: headline metrics + the details page
# usage: bash tools/ncu_full_txt.sh report.ncu-rep > profiles/<name>.txt
python tools/ncu_summary.py "$1"
ncu -i "$1" --page details --csv 2>/dev/null | python -c '
import csv, sys
rows = list(csv.reader(sys.stdin))
h = rows[0]
si, mi, ui, vi = (h.index("Section Name"), h.index("Metric Name"),
                  h.index("Metric Unit"), h.index("Metric Value"))
for r in rows[1:]:
    print(f"{r[si]:34s} {r[mi]:50s} {r[vi]:>14s} {r[ui]}")
'
