"""CPU tests of bench.py's input builder: the c5-shaped multi-day blob (day k = seed + k, date + k,
same journey ids) is the concatenation of the per-day generator outputs with shifted shard
offsets, and every shard starts with the header."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def test_multi_day_generate_matches_per_day_generator():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2305_07454_b200 import synth_day
    blob, offs, rows = bench.generate(50, 3, 120.0, seed=4, days=3)
    assert len(offs) == 3 * 3 + 1 and offs[0] == 0 and offs[-1] == len(blob)
    assert all(b >= a for a, b in zip(offs, offs[1:]))
    total = 0
    for k, day in enumerate(("2021-05-09", "2021-05-10", "2021-05-11")):
        b, o, r = synth_day(seed=4 + k, journeys=50, shards=3, mean_duration=120.0, day=day)
        total += r
        for i in range(3):
            got = blob[offs[3 * k + i]:offs[3 * k + i + 1]]
            exp = b[o[i]:o[i + 1]]
            assert np.array_equal(got, exp)
            assert bytes(got[:10]) == b"Journey Id"
            if len(got) > 200:
                assert day.encode() in bytes(got[:200])
    assert rows == total


def test_single_day_generate_is_the_generator():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2305_07454_b200 import synth_day
    blob, offs, rows = bench.generate(40, 2, 100.0, seed=9)
    b, o, r = synth_day(seed=9, journeys=40, shards=2, mean_duration=100.0)
    assert np.array_equal(blob, b) and list(offs) == list(o) and rows == r
