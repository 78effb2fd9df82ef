"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck): decode fast
and full-sort paths, dictionary, radix sorts, fold (journey lanes with windows + spill, and
(journey, bin) groups), finalize, routing and the multi-GPU combine, and the records entry
point. Diagnostics, not product."""
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402

import paper_2305_07454_b200 as cvlg  # noqa: E402
from helpers import commuter_days, malformed_contents, shuffle_rows, write_shards  # noqa: E402

with tempfile.TemporaryDirectory() as d:
    d = Path(d)
    cvlg.cvlg.synth_write_day(d / "day", seed=5, journeys=40, shards=4, mean_duration=200.0)
    day = sorted(str(p) for p in (d / "day").glob("*.csv"))
    sets = {
        "synth": (day, cvlg.GridSpec()),
        "shuffled": (shuffle_rows(day, d / "shuf", 3, 1), cvlg.GridSpec()),
        "malformed": (write_shards(d / "bad", malformed_contents(3)), cvlg.GridSpec()),
        "multiday_fine": (write_shards(d / "md", commuter_days(40, 2, 14, seed=1)),
                          cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1)),
    }
    ctx = cvlg.Context()
    m = cvlg.MultiGPU([0, 0])
    for name, (paths, spec) in sets.items():
        a = cvlg.run_pipeline(paths, spec, ctx=ctx)  # few journeys: bin-group fold
        os.environ["CVLG_FOLD_GROUPS"] = "0"  # journey lanes (+ windows)
        c = cvlg.run_pipeline(paths, spec, ctx=ctx)
        del os.environ["CVLG_FOLD_GROUPS"]
        b = m.run_pipeline(paths, spec)
        assert np.array_equal(a.planes, b.planes) and np.array_equal(a.planes, c.planes), name
        print(name, "ok", int(a.volume.sum()))
    # records entry point (run_pipeline_from_records), with a duplicate and a conflict
    import datetime
    recs = []
    for s_i, path in enumerate(day):
        lines = Path(path).read_bytes().split(b"\n")[1:]
        for ln, line in enumerate(lines, start=1):
            if not line:
                continue
            f = line.split(b",")
            t = datetime.datetime.strptime(f[1].decode(), "%Y-%m-%d %H:%M:%S")
            ts = int((t - datetime.datetime(1970, 1, 1)).total_seconds())
            recs.append((f[0], ts, float(f[2]), float(f[3]), f[4], float(f[5]), float(f[6]),
                         path.encode(), ln))
    recs.append(recs[5][:5] + (recs[5][5] + 1.0,) + recs[5][6:7] + (b"/z.csv", 1))
    recs.append(recs[9][:7] + (b"/a.csv", 2))
    r = cvlg.run_pipeline_from_records(recs, cvlg.GridSpec(), ctx=ctx)
    print("records ok", int(r.volume.sum()))
