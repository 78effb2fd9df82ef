"""Top source lines by executed warp-instructions for one file of an ncu report.
   python tools/ncu_top_lines.py report.ncu-rep kernel-regex file [top]"""
import csv
import io
import subprocess
import sys

rep, kern, fname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
cur = hdr = None
rows = []
num = lambda x: int(x) if x.strip().lstrip('-').isdigit() else 0
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if cur == fname and hdr and r and r[0].isdigit() and len(r) > 8:
        rows.append((num(r[7]), num(r[4]), int(r[0]), r[1][:100]))
for i, s, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{i / 1e6:8.1f}M stall {s:6d} {fname}:{ln} {src}")
