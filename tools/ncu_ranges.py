"""Sum ncu source-level warp-instructions over line ranges (phases) of the decode kernel.
   python tools/ncu_ranges.py report.ncu-rep kernel-regex"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
cur = hdr = None
per = {}
num = lambda x: int(x) if x.strip().lstrip('-').isdigit() else 0
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and len(r) > 8:
        per[(cur, int(r[0]))] = per.get((cur, int(r[0])), 0) + num(r[7])
ranges = [a.split(":") for a in sys.argv[3:]]
tot = sum(per.values())
acc = 0
for name, f, lo, hi in ranges:
    s = sum(v for (ff, ln), v in per.items() if ff == f and int(lo) <= ln <= int(hi))
    acc += s
    print(f"{name:28s} {s / 1e6:8.1f}M {100 * s / tot:5.1f}%")
print(f"{'other':28s} {(tot - acc) / 1e6:8.1f}M {100 * (tot - acc) / tot:5.1f}%   total {tot / 1e6:.1f}M")
