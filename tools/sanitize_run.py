"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck): decode fast
and full-sort paths, dictionary, radix sorts, fold (windows + spill), finalize, routing and the
multi-GPU combine. Diagnostics, not product."""
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
        a = cvlg.run_pipeline(paths, spec, ctx=ctx)
        b = m.run_pipeline(paths, spec)
        assert np.array_equal(a.planes, b.planes), name
        print(name, "ok", int(a.volume.sum()))
