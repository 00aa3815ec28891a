"""Executed-instruction mix of one kernel by SASS opcode from a full ncu
capture: python tools/ncu_opcodes.py report.ncu-rep kernel_regex units"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ii, si = h.index("Instructions Executed"), h.index("Source")
cnt, tot = collections.Counter(), 0
for r in rows[2:]:
    try:
        n = int(r[ii])
    except (ValueError, IndexError):
        continue
    f = r[si].split()
    if not f:
        continue
    op = f[1] if f[0].startswith("@") else f[0]
    cnt[op.split(".")[0]] += n
    tot += n
print(f"total {tot}  per unit {tot / units:.1f}")
for op, n in cnt.most_common(30):
    print(f"{op:10s} {100 * n / tot:5.1f}%  {n / units:8.1f}")
