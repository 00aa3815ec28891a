"""Summarise an ncu report (run here, no GPU needed):
python tools/ncu_summary.py gpurun_out/prof_step.ncu-rep [launch_index]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2 + idx]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "lts__t_sector_hit_rate.pct", "launch__grid_size"]
for w in want:
    for h, u, v in zip(hdr, units, vals):
        if h == w:
            print(f"{w:70s} {v} {u}")
st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), num(v))
      for h, v in zip(hdr, vals)
      if "pcsamp_warps_issue_stalled" in h and num(v) is not None
      and not h.endswith("not_issued")]
tot = sum(v for _, v in st) or 1
print("stall samples:", ", ".join(f"{h} {100*v/tot:.0f}%"
                                  for h, v in sorted(st, key=lambda x: -x[1])[:8]))
