"""Quick GPU-vs-reference diff on a small synthetic day (debug aid)."""
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_2305_07454_b200 as cvlg  # noqa: E402
from oracle.oracle import Ref  # noqa: E402
from helpers import diff_lattice, stats_dict  # noqa: E402

ref = Ref()
with tempfile.TemporaryDirectory() as d:
    ref.generate_day(d, seed=1, journeys=int(sys.argv[1]) if len(sys.argv) > 1 else 20, shards=2)
    paths = sorted(str(p) for p in Path(d).glob("*.csv"))
    for spec in [cvlg.GridSpec(), cvlg.GridSpec(lat_step=10, lon_step=10)]:
        ep, er, est, _ = ref.run_pipeline(paths, spec)
        st = cvlg.PipelineStats()
        try:
            lat = cvlg.run_pipeline(paths, spec, stats=st)
            print("diff:", diff_lattice(ep, er, lat.planes, lat.raw) or "none")
        except Exception as e:
            print("error:", e)
        print("ref ", est)
        print("ours", stats_dict(st))
