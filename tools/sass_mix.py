"""Executed warp instructions per SASS opcode (and per pipe class) from
`ncu -i rep --page source --csv --print-source sass -k regex:K > sass.csv`.
   python tools/sass_mix.py sass.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = hdr.index("Instructions Executed")
cnt = collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ix or not r[ix].strip().isdigit():
        continue
    src = r[1].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1] if " " in src else src
    op = src.split()[0].rstrip(";") if src else "?"
    n = int(r[ix])
    cnt[op] += n
    tot += n
base = collections.Counter()
for op, n in cnt.items():
    base[op.split(".")[0]] += n
print(f"total {tot / 1e6:.1f}M warp instructions")
for op, n in base.most_common(top):
    print(f"{op:12s} {n / 1e6:8.1f}M {100 * n / tot:5.1f}%")
