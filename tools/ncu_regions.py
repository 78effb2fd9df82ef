"""Group ncu source-level instruction counts / stall samples by code region: device functions
and '// ---- ' phase markers are detected from the captured source text.
   python tools/ncu_regions.py report.ncu-rep kernel-regex"""
import csv
import io
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fn_re = re.compile(r"^(?:template.*)?(?:static\s+)?(?:CVLG_HD\w*|__device__|__global__|__host__)[^(]*?\b(\w+)\s*\(")
cur = None
hdr = None
label = "?"
agg = {}
tot_i = tot_s = 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        label = cur
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] != "" and len(r) >= 2:
        src = r[1]
        m = fn_re.match(src.strip())
        if m:
            label = f"{cur}:{m.group(1)}"
        elif src.strip().startswith("// ---- "):
            label = f"{cur}:{src.strip()[8:60]}"
        try:
            inst, samp = int(r[7] or 0), int(r[4] or 0)
        except (ValueError, IndexError):
            continue
        a = agg.setdefault(label, [0, 0])
        a[0] += inst
        a[1] += samp
        tot_i += inst
        tot_s += samp
print(f"{'region':64s} {'warp-inst':>10s} {'inst%':>6s} {'stall%':>6s}")
for k, (i, s) in sorted(agg.items(), key=lambda x: -x[1][0]):
    if i or s:
        print(f"{k[:64]:64s} {i / 1e6:9.1f}M {100 * i / tot_i:5.1f}% {100 * s / tot_s:5.1f}%")
print(f"{'TOTAL':64s} {tot_i / 1e6:9.1f}M")
