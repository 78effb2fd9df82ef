"""Ingest ring geometry sweep (diagnostics, not product): cvlg_run_pipeline(paths) end to end on
the c2 shard files with CVLG_RING_MB / CVLG_RING_SLOTS / reader-thread overrides.
  python tools/ring_sweep.py [--journeys N] [--reps R]"""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_07454_b200 as cvlg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--journeys", type=int, default=100_000)
ap.add_argument("--shards", type=int, default=128)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--dir", default="/tmp/cvlg_probe")
ap.add_argument("--grid", default="2:64,4:32,8:16,16:16,32:16,64:8,4:64")
ap.add_argument("--threads", default="")
a = ap.parse_args()
d = Path(a.dir) / f"j{a.journeys}"
if not (d / "done").exists():
    cvlg.cvlg.synth_write_day(d, seed=1, journeys=a.journeys, shards=a.shards, mean_duration=500.0)
    (d / "done").write_text("1")
paths = sorted(str(p) for p in d.glob("shard_*.csv"))
total = sum(os.path.getsize(p) for p in paths)
T = os.cpu_count()
print(f"{len(paths)} files, {total / 1e9:.2f} GB, cpu_count {T}", flush=True)
spec = cvlg.GridSpec()
Td, _, R, C = spec.dims()
planes = np.empty((Td, 8, R, C), dtype=np.uint32)
raw = np.empty((Td, 4, R, C), dtype=np.uint32)
cvlg.pin_host(planes)
cvlg.pin_host(raw)
ctx = cvlg.Context(0)
threads = [int(x) for x in a.threads.split(",")] if a.threads else [T]
for g in a.grid.split(","):
    mb, slots = g.split(":")
    os.environ["CVLG_RING_MB"] = mb
    os.environ["CVLG_RING_SLOTS"] = slots
    for nt in threads:
        os.environ["CVLG_RING_READERS"] = str(nt)
        cvlg.run_pipeline(paths, spec, n_threads=T, ctx=ctx, out=(planes, raw))
        ts = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cvlg.run_pipeline(paths, spec, n_threads=T, ctx=ctx, out=(planes, raw))
            ts.append(time.perf_counter() - t0)
        best = min(ts)
        print(f"ring {mb:>3} MB x {slots:>3} slots, {nt:2d} readers: best {1000 * best:7.1f} ms "
              f"= {total / best / 1e9:5.1f} GB/s (median {1000 * sorted(ts)[len(ts) // 2]:7.1f} ms)",
              flush=True)
