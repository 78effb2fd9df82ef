"""Runs the device-resident pipeline on the c2 workload for ncu captures:
    ncu ... python tools/profile_step.py [--journeys N] [--steps S]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2305_07454_b200 as cvlg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--journeys", type=int, default=100_000)
ap.add_argument("--shards", type=int, default=16)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--shuffle", action="store_true")
ap.add_argument("--days", type=int, default=1)
ap.add_argument("--fine", action="store_true")
ap.add_argument("--mean-duration", type=float, default=500.0)
ap.add_argument("--print-csv-bytes", action="store_true")
a = ap.parse_args()
if a.days > 1:  # c5 shape: day k uses seed 1 + k and date + k; its shards follow day k-1's
    import datetime
    import numpy as np
    blobs, offs, rows = [], [0], 0
    for k in range(a.days):
        d = (datetime.date(2021, 5, 9) + datetime.timedelta(days=k)).isoformat()
        b, o, r = cvlg.synth_day(seed=1 + k, journeys=a.journeys, shards=a.shards,
                                 mean_duration=500.0, day=d)
        b0 = offs[-1]
        offs.extend(b0 + int(x) for x in o[1:])
        blobs.append(b)
        rows += r
    blob = np.concatenate(blobs)
else:
    blob, offs, rows = cvlg.synth_day(seed=1, journeys=a.journeys, shards=a.shards,
                                      mean_duration=a.mean_duration)
if a.shuffle:  # adversarial variant: the full-sort path
    blob, offs = cvlg.cvlg.shuffle_rows(blob, offs, a.shards, seed=7)
if a.print_csv_bytes:
    print("csv_bytes", int(offs[-1]), flush=True)
spec = cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1) if a.fine else cvlg.GridSpec()
T, _, R, C = spec.dims()
d_csv = torch.from_numpy(blob).cuda()
d_planes = torch.empty((T, 8, R, C), dtype=torch.int32, device="cuda")
d_raw = torch.empty((T, 4, R, C), dtype=torch.int32, device="cuda")
ctx = cvlg.Context()
times = []
for _ in range(a.steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cvlg.run_pipeline_device(d_csv.data_ptr(), offs, d_planes.data_ptr(), d_raw.data_ptr(), spec,
                             ctx=ctx, stream=torch.cuda.current_stream().cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
print("rows", rows, "stage_ms", ctx.stage_ms(), "step_ms", ["%.2f" % t for t in times])
