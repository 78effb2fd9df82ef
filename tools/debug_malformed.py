"""Reproduce tests/test_gpu_parity.py::test_malformed_and_edge_inputs and print the divergence
(stats + the differing cell's reference records). Debug aid."""
import random
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_2305_07454_b200 as cvlg  # noqa: E402
import corpus  # noqa: E402
from oracle.oracle import Ref  # noqa: E402
from helpers import HEADER, diff_lattice, stats_dict, write_shards  # noqa: E402

ref = Ref()
rng = random.Random(5)
body = corpus.line_corpus(rng, 3000)
good = [b"jj%03d,2021-05-09 %02d:%02d:%02d,%.6f,%.6f,65101,%.2f,%.2f" % (
    i % 17, (i // 3600) % 24, (i // 60) % 60, i % 60, 36.1 + (i % 400) * 0.01,
    -95.7 + (i % 600) * 0.011, (i * 7.3) % 140, (i * 13.7) % 360) for i in range(4000)]
mixed = body + good
rng.shuffle(mixed)
contents = [
    HEADER + b"\r\n" + b"\r\n".join(mixed[:1500]) + b"\r\n",
    HEADER + b"\n" + b"\n\n".join(mixed[1500:4000]),
    b"",
    b"nope,nope\n1,2\n",
    b"heading,speed,zip code,longitude,latitude,timestamp,journey-id\n" + b"\n".join(
        b"%s,%s,%s,%s,%s,%s,%s" % tuple(reversed(l.split(b",")[:7])) for l in good[:800]
        if len(l.split(b",")) == 7),
    HEADER,
    HEADER + b"\n" + b"\n".join(mixed[4000:]) + b"\n",
]
with tempfile.TemporaryDirectory() as d:
    paths = write_shards(Path(d), contents)
    spec = cvlg.GridSpec()
    ep, er, est, _ = ref.run_pipeline(paths, spec, None, n_partitions=3, n_threads=1)
    st = cvlg.PipelineStats()
    lat = cvlg.run_pipeline(paths, spec, stats=st)
    print("diff:", diff_lattice(ep, er, lat.planes, lat.raw) or "none")
    print("ref ", est)
    print("ours", stats_dict(st))
    # lines that land in differing volume cells
    vd = np.argwhere(ep[:, 4:8] != lat.planes[:, 4:8])
    print("volume diffs:", vd[:10].tolist())
    for k, c in enumerate(contents):
        for j, line in enumerate(c.split(b"\n")):
            if b"12:00:00" in line:
                print(k, j, line)
