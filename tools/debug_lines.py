"""Per-line GPU-vs-reference check of the malformed-input corpus (debug aid): every corpus line
alone in a shard (LF and CRLF endings); prints the lines whose stats or lattice differ."""
import random
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_2305_07454_b200 as cvlg  # noqa: E402
import corpus  # noqa: E402
from oracle.oracle import Ref  # noqa: E402
from helpers import HEADER, diff_lattice, stats_dict, write_shards  # noqa: E402

ref = Ref()
rng = random.Random(5)
body = corpus.line_corpus(rng, 3000)
bad = 0
with tempfile.TemporaryDirectory() as d:
    for i, line in enumerate(body):
        for eol in (b"\n", b"\r\n"):
            paths = write_shards(Path(d) / f"c{i}_{len(eol)}", [HEADER + eol + line + eol + line + eol])
            spec = cvlg.GridSpec()
            ep, er, est, _ = ref.run_pipeline(paths, spec, None, n_partitions=1, n_threads=1)
            st = cvlg.PipelineStats()
            lat = cvlg.run_pipeline(paths, spec, stats=st)
            dd = diff_lattice(ep, er, lat.planes, lat.raw)
            if dd or stats_dict(st) != est:
                bad += 1
                if bad < 20:
                    print(repr(line), eol, dd, "\n  ref ", est, "\n  ours", stats_dict(st))
print("lines", len(body), "bad", bad)
