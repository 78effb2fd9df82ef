"""Summarise an ncu report: key metrics, stall reasons, source hot spots.
   python tools/ncu_summary.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv", "-k", f"regex:{kern}"))))
if len(raw) > 2:
    h = raw[0]
    for row in raw[2:]:
        d = dict(zip(h, row))
        print("==", d.get("Kernel Name", "")[:80])
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__warps_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "launch__occupancy_limit_registers",
                "launch__occupancy_limit_shared_mem", "sm__inst_executed.sum",
                "smsp__thread_inst_executed_per_inst_executed.ratio",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
        for k in keys:
            if k in d:
                print(f"  {k:70s} {d[k]}")
        stalls = [(k, d[k]) for k in h if k.startswith("smsp__average_warp_latency_issue_stalled")
                  or k.startswith("smsp__pcsamp_warps_issue_stalled_")]
        vals = []
        for k, v in stalls:
            try:
                vals.append((float(v.replace(",", "")), k))
            except ValueError:
                pass
        for v, k in sorted(vals, reverse=True)[:12]:
            print(f"  {k:70s} {v}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass",
                                          "-k", f"regex:{kern}"))))
cur = None
hdr = None
out = []
for r in src:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] != "" and len(r) > 8:
        try:
            out.append((int(r[4] or 0), int(r[7] or 0), cur, r[0], r[1][:90]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out)
print("source: samples", tot, "warp-inst", ti)
for o in sorted(out, reverse=True)[:top]:
    print(f"{100 * o[0] / tot:5.1f}% inst={o[1] / 1e6:8.1f}M {o[2]}:{o[3]} {o[4]}")
