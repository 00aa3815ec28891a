"""Per-source-line instruction counts and stall samples of one kernel from a
full ncu capture (compiled with -lineinfo, captured with --import-source on).
usage: python tools/ncu_src_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")])
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    if ie or st:
        rows.append((ie, st, fname, r[0], r[1].strip()[:90]))
tot_i = sum(x[0] for x in rows) or 1
tot_s = sum(x[1] for x in rows) or 1
print(f"total inst {tot_i}  stall samples {tot_s}")
for key, name in ((0, "instructions"), (1, "stall samples")):
    print(f"--- top lines by {name}")
    for ie, st, f, ln, src in sorted(rows, key=lambda x: -x[key])[:top]:
        print(f"{100*ie/tot_i:5.1f}% {100*st/tot_s:5.1f}%  {f}:{ln}  {src}")
