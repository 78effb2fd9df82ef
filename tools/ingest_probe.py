"""Where does the e2e time go? (diagnostics, not product)
  python tools/ingest_probe.py [--journeys N] [--threads T]
1. pread of the shard files (page cache) into pinned memory with T threads (no H2D)
2. H2D of pinned 32 MB chunks on one stream (no reads)
3. cvlg_run_pipeline(paths) end to end, with CVLG_TRACE phase times"""
import argparse
import os
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2305_07454_b200 as cvlg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--journeys", type=int, default=100_000)
ap.add_argument("--shards", type=int, default=128)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--dir", default="/tmp/cvlg_probe")
a = ap.parse_args()
T = a.threads or os.cpu_count()
d = Path(a.dir) / f"j{a.journeys}"
if not (d / "done").exists():
    t0 = time.perf_counter()
    cvlg.cvlg.synth_write_day(d, seed=1, journeys=a.journeys, shards=a.shards, mean_duration=500.0)
    (d / "done").write_text("1")
    print(f"generated in {time.perf_counter() - t0:.1f} s")
paths = sorted(str(p) for p in d.glob("shard_*.csv"))
total = sum(os.path.getsize(p) for p in paths)
print(f"{len(paths)} files, {total / 1e9:.2f} GB, {T} threads")

CH = 32 << 20
ring = torch.empty(16 * CH, dtype=torch.uint8).pin_memory()
rnp = ring.numpy()


def read_all(nthreads):
    chunks = [(p, o, min(CH, os.path.getsize(p) - o)) for p in paths for o in range(0, os.path.getsize(p), CH)]
    nxt = [0]
    lock = threading.Lock()

    def work(slot):
        while True:
            with lock:
                k = nxt[0]
                nxt[0] += 1
            if k >= len(chunks):
                return
            p, o, n = chunks[k]
            fd = os.open(p, os.O_RDONLY)
            mv = memoryview(rnp[slot * CH: slot * CH + n])
            got = 0
            while got < n:
                got += os.preadv(fd, [mv[got:]], o + got)
            os.close(fd)
    th = [threading.Thread(target=work, args=(i % 16,)) for i in range(nthreads)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    return time.perf_counter() - t0


read_all(T)
for nt in sorted({4, 8, T}):
    dt = read_all(nt)
    print(f"1. pread page cache -> pinned, {nt:2d} threads: {total / dt / 1e9:6.1f} GB/s")

dev = torch.empty(total + 64, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        off = 0
        while off < total:
            n = min(CH, total - off)
            k = (off // CH) % 16
            dev[off: off + n].copy_(ring[k * CH: k * CH + n], non_blocking=True)
            off += n
    s.synchronize()
    dt = time.perf_counter() - t0
print(f"2. H2D pinned 32 MB chunks, one stream: {total / dt / 1e9:6.1f} GB/s ({dt * 1e3:.1f} ms)")

ctx = cvlg.Context()
st = cvlg.PipelineStats()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cvlg.run_pipeline(paths, cvlg.GridSpec(), n_threads=T, stats=st, ctx=ctx)
    dt = time.perf_counter() - t0
    print(f"3. cvlg_run_pipeline(paths): {dt * 1e3:.1f} ms = {total / dt / 1e9:.1f} GB/s input, "
          f"device stages {ctx.stage_ms()}")
os.environ["CVLG_TRACE"] = "1"
cvlg.run_pipeline(paths, cvlg.GridSpec(), n_threads=T, stats=st, ctx=ctx)
