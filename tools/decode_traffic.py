"""Writes profiles/decode_traffic.json: K1's DRAM bytes per launch (one ncu capture per workload)
for bench.py's roofline `traffic` field.  Run on the GPU box:
    python tools/decode_traffic.py c2 c3"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
WL = {"c2": 100_000, "c3": 1_000_000}
out = ROOT / "profiles" / "decode_traffic.json"
entries = json.loads(out.read_text()) if out.exists() else []
if isinstance(entries, dict):
    entries = [entries]
for name in sys.argv[1:]:
    r = subprocess.run(["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
                        "--clock-control", "none", "-k", "regex:decode_kernel", "-c", "1", "--csv",
                        sys.executable, str(ROOT / "tools" / "profile_step.py"), "--journeys", str(WL[name]),
                        "--shards", "128", "--steps", "1", "--print-csv-bytes"],
                       capture_output=True, text=True)
    m, csv_bytes = {}, None
    for line in r.stdout.splitlines():
        if line.startswith("csv_bytes "):
            csv_bytes = int(line.split()[1])
    for row in csv.reader(io.StringIO("\n".join(l for l in r.stdout.splitlines() if l.startswith('"')))):
        if len(row) > 14 and row[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            unit, v = row[13], float(row[14].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
            m[row[12]] = v * scale
    if not m or csv_bytes is None:
        print(r.stdout[-3000:], r.stderr[-3000:])
        continue
    e = {"kernel": "decode_kernel", "workload": f"{name} ({WL[name]} journeys, 128 shards)",
         "csv_bytes": csv_bytes, "dram_read": int(m["dram__bytes_read.sum"]),
         "dram_write": int(m["dram__bytes_write.sum"]),
         "dram_bytes_per_launch": int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]),
         "ncu_ns": m.get("gpu__time_duration.sum"), "source": "ncu --metrics dram__bytes_{read,write}.sum (tools/decode_traffic.py)"}
    entries = [x for x in entries if x.get("csv_bytes") != csv_bytes] + [e]
    print(json.dumps(e))
out.write_text(json.dumps(entries, indent=1))
