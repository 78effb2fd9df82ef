"""Key metrics + stall samples + top source lines of one kernel in an ncu --set full report.
   python tools/ncu_summary.py report.ncu-rep kernel-regex source-file [top]"""
import csv
import io
import subprocess
import sys

rep, kern, src = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
name = v[h.index("Kernel Name")] if "Kernel Name" in h else kern
print(f"== {name}")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
for k in want:
    if k in h:
        print(f"  {k:70s} {v[h.index(k)]} {rows[1][h.index(k)]}")
st = [(float(x.replace(',', '')), k) for k, x in zip(h, v)
      if k.startswith("smsp__pcsamp_warps_issue_stalled") and "not_issued" not in k and x]
for x, k in sorted(st, reverse=True)[:8]:
    print(f"  {k:70s} {int(x)}")
out = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_top_lines.py"), rep, kern,
                      src, str(top)], capture_output=True, text=True).stdout
print(f"source {src}: top lines by executed warp instructions")
print(out, end="")
