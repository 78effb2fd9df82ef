"""Full-c3 parity check (evidence, not a test: ~1-2 min of 16-core reference time and tens of GB
of host memory): the bench's c3 shard files (1,000,000 journeys, ~499M rows) through
cvlg_run_pipeline on the GPU and through the UNMODIFIED reference cvl::run_pipeline
(oracle/_ref) in a child process whose address space is capped (RLIMIT_AS), so running out of
host memory fails the child instead of the box. Prints one JSON line.
    python tools/c3_parity.py [--data-dir /tmp/cvlg_bench] [--as-gb 170]"""
import argparse
import hashlib
import json
import os
import resource
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def sha(planes, raw):
    import numpy as np
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(planes).view(np.uint8))
    h.update(np.ascontiguousarray(raw).view(np.uint8))
    return h.hexdigest()


def child(paths_file, out_file):
    from oracle.oracle import Ref

    class Spec:
        lat_min, lat_max, lon_min, lon_max = 36.0, 40.6, -95.8, -89.1
        lat_step = lon_step = 0.1
        min_step, dxn_step, dxn_offset = 5, 90, 0.0
    paths = json.loads(Path(paths_file).read_text())
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    planes, raw, st, _ = Ref().run_pipeline(paths, Spec, None, n_partitions=2 * threads,
                                            n_threads=threads, raw=True)
    dt = time.perf_counter() - t0
    Path(out_file).write_text(json.dumps({"sha": sha(planes, raw), "stats": st, "seconds": dt,
                                          "threads": threads}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--data-dir", default="/tmp/cvlg_bench")
    ap.add_argument("--as-gb", type=float, default=170.0)
    ap.add_argument("--child", nargs=2)
    a = ap.parse_args()
    if a.child:
        child(*a.child)
        return
    import bench
    args = argparse.Namespace(workload="c3", data_dir=a.data_dir, threads=0)
    paths, man, _ = bench.ensure_dataset(args, bench.our_generator(os.cpu_count() or 1))
    import paper_2305_07454_b200 as cvlg
    st = cvlg.PipelineStats()
    t0 = time.perf_counter()
    lat = cvlg.run_pipeline(paths, cvlg.GridSpec(), stats=st)
    gpu_s = time.perf_counter() - t0
    ours = {"sha": sha(lat.planes, lat.raw), "rows_read": st.rows_read, "parsed": st.parsed,
            "accepted": st.accepted, "duplicates_dropped": st.duplicates_dropped}
    del lat
    pf, of = Path("/tmp/c3_paths.json"), Path("/tmp/c3_ref.json")
    pf.write_text(json.dumps(paths))
    of.unlink(missing_ok=True)
    lim = int(a.as_gb * (1 << 30))

    def cap():
        resource.setrlimit(resource.RLIMIT_AS, (lim, lim))
    rc = subprocess.call([sys.executable, __file__, "--child", str(pf), str(of)], preexec_fn=cap)
    ref = json.loads(of.read_text()) if rc == 0 and of.exists() else None
    line = {"workload": "c3 (1,000,000 journeys, seed 1, 128 shard files)", "rows": man["rows"],
            "ours": ours, "ours_seconds_first_call": round(gpu_s, 2),
            "reference": ref, "reference_rc": rc}
    if ref:
        rs = ref["stats"]
        line["lattice_and_stats_bit_identical"] = bool(
            ref["sha"] == ours["sha"] and rs["rows_read"] == ours["rows_read"]
            and rs["parsed"] == ours["parsed"] and rs["accepted"] == ours["accepted"]
            and rs["duplicates_dropped"] == ours["duplicates_dropped"])
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
