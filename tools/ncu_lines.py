"""Per-source-line / per-line-range instruction and stall totals from an ncu report.
   python tools/ncu_lines.py report.ncu-rep kernel-regex file.cu a-b:name [a-b:name ...]"""
import csv
import io
import subprocess
import sys

rep, kern, fname = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
cur = hdr = None
agg = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and len(r) > 8:
        num = lambda x: int(x) if x.strip().lstrip('-').isdigit() else 0
        agg[(cur, int(r[0]))] = (num(r[4]), num(r[7]))
ti = sum(v[1] for v in agg.values()) or 1
ts = sum(v[0] for v in agg.values()) or 1
print(f"total warp-inst {ti / 1e6:.1f}M samples {ts}")
for f in sorted({k[0] for k in agg}):
    i = sum(v[1] for k, v in agg.items() if k[0] == f)
    s = sum(v[0] for k, v in agg.items() if k[0] == f)
    print(f"  {f:30s} {i / 1e6:9.1f}M {100 * i / ti:5.1f}%  stall {100 * s / ts:5.1f}%")
for spec in sys.argv[4:]:
    rng, name = spec.split(":", 1)
    a, b = map(int, rng.split("-"))
    i = sum(v[1] for k, v in agg.items() if k[0] == fname and a <= k[1] <= b)
    s = sum(v[0] for k, v in agg.items() if k[0] == fname and a <= k[1] <= b)
    print(f"  {name:30s} {i / 1e6:9.1f}M {100 * i / ti:5.1f}%  stall {100 * s / ts:5.1f}%")
