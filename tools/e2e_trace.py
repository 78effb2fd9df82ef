"""c3 e2e timeline (diagnostics): cvlg_run_pipeline(paths) on the bench's c3 shard files with
CVLG_TRACE=1 (phase timestamps on stderr) after two warm-up calls.
    CVLG_TRACE=1 python tools/e2e_trace.py"""
import argparse
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2305_07454_b200 as cvlg  # noqa: E402

args = argparse.Namespace(workload="c3", data_dir="/tmp/cvlg_bench", threads=0)
paths, man, _ = bench.ensure_dataset(args, bench.our_generator(os.cpu_count() or 1))
spec = cvlg.GridSpec()
T, _, R, C = spec.dims()
planes = np.empty((T, 8, R, C), dtype=np.uint32)
raw = np.empty((T, 4, R, C), dtype=np.uint32)
cvlg.pin_host(planes)
cvlg.pin_host(raw)
ctx = cvlg.Context(0)
trace = os.environ.pop("CVLG_TRACE", None)
for _ in range(2):
    cvlg.run_pipeline(paths, spec, n_partitions=32, n_threads=os.cpu_count(), ctx=ctx, out=(planes, raw))
if trace:
    os.environ["CVLG_TRACE"] = trace
t0 = time.perf_counter()
cvlg.run_pipeline(paths, spec, n_partitions=32, n_threads=os.cpu_count(), ctx=ctx, out=(planes, raw))
print(f"e2e {1000 * (time.perf_counter() - t0):.1f} ms", flush=True)
