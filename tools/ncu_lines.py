"""Per-source-line instruction / stall breakdown of an ncu report:
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
cur, hdr, agg, fn = None, None, {}, None
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "Function Name":
        if fn is not None and r[1] != fn:
            break  # first kernel only
        fn = r[1]
        continue
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        ex, stl = int(r[7]), int(r[4])
    except ValueError:
        continue
    k = (cur, int(r[0]), r[1].strip()[:80])
    e = agg.setdefault(k, [0, 0])
    e[0] += ex
    e[1] += stl
tot = sum(v[0] for v in agg.values()) or 1
tst = sum(v[1] for v in agg.values()) or 1
print(f"instructions {tot}  stall samples {tst}")
for (f, ln, src), (ex, stl) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*ex/tot:5.1f}% st{100*stl/tst:5.1f}% {f}:{ln} {src}")
