"""Summarise an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes]) per kernel.
   python tools/launch_summary.py launches.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
idi = h.index("ID")
per = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    key = (r[idi], r[ki])
    per.setdefault(key, {})[r[mi]] = float(r[vi].replace(",", ""))
tot = {}
for (lid, name), m in per.items():
    n = name.split("(")[0].replace("(anonymous namespace)::", "").replace("cvlg::", "")[:48]
    t = tot.setdefault(n, [0.0, 0, 0.0])
    t[0] += m.get("gpu__time_duration.sum", 0.0)
    t[1] += 1
    t[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
s = sum(v[0] for v in tot.values())
print(f"{'kernel':50s} {'ms':>9s} {'share':>6s} {'launches':>8s} {'DRAM GB':>8s} {'GB/s':>8s}")
for n, (t, c, b) in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"{n:50s} {t / 1e6:9.3f} {100 * t / s:5.1f}% {c:8d} {b / 1e9:8.3f} {b / t:8.1f}")
print(f"{'TOTAL':50s} {s / 1e6:9.3f}")
