"""Per-journey feature table (csrc/features.cu; north_star extension).

NOT IN THE REFERENCE: there is no reference function, test or golden vector for these columns,
so parity is UNPINNED against the reference. The GPU results are checked against this repo's CPU
restatement (tests/features_oracle.py), whose record set comes from the reference's own parser
and whose formulas are checked here on hand-computed traces. Tolerances: integer columns, epoch
seconds, max_speed and dwell_s exact; length_m / max_step_m / max_abs_accel within 1e-12
relative (CUDA's sin/cos/asin vs the host libm may differ in the last ulp)."""
from __future__ import annotations

import math
import random
from pathlib import Path

import numpy as np
import pytest

import features_oracle as fo
from helpers import HEADER, shuffle_rows
from test_hostparse import hp  # noqa: F401  (fixture)


def test_restatement_known_answers():
    # 1 degree of longitude on the equator = R * pi / 180
    assert fo.haversine_m(0.0, 0.0, 0.0, 1.0) == pytest.approx(6371008.8 * math.pi / 180, rel=1e-15)
    assert fo.haversine_m(37.0, -92.0, 37.0, -92.0) == 0.0
    # stop episodes / dwell / acceleration on a 4-point trace (stop_speed 5)
    f = fo.journey_features([(0, 0.0, 0.0, 0.0), (10, 0.0, 0.0, 0.0), (20, 0.0, 0.001, 10.0),
                             (30, 0.0, 0.001, 0.0)], 5.0)
    assert f["points"] == 4 and f["t_first"] == 0 and f["t_last"] == 30
    assert f["stops"] == 2 and f["dwell_s"] == 10.0 and f["max_abs_accel"] == 1.0
    assert f["max_speed"] == 10.0
    assert f["length_m"] == pytest.approx(6371008.8 * math.pi / 180 * 0.001, rel=1e-9)


def _compare(rows, feats, ids):
    assert len(rows) == len(ids) == len(feats["points"])
    for i, (jid, f) in enumerate(rows):
        assert ids[i] == jid, (i, ids[i], jid)
        for k in ("points", "t_first", "t_last", "stops"):
            assert int(feats[k][i]) == f[k], (jid, k, feats[k][i], f[k])
        for k in ("max_speed", "dwell_s"):
            assert float(feats[k][i]) == f[k], (jid, k, feats[k][i], f[k])
        for k in ("length_m", "max_step_m", "max_abs_accel"):
            assert float(feats[k][i]) == pytest.approx(f[k], rel=1e-12, abs=1e-9), (jid, k)


def _shards(paths):
    return [Path(p).read_bytes() for p in paths]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["synth", "shuffled", "dups_filters"])
def test_features_vs_restatement(ref, hp, tmp_path, variant):
    import paper_2305_07454_b200 as cvlg
    d = tmp_path / "day"
    ref.generate_day(str(d), seed=5, journeys=40, shards=4, mean_duration=200.0,
                     sample_period=0.5 if variant == "dups_filters" else 1.0)
    paths = sorted(str(p) for p in d.glob("*.csv"))
    if variant == "shuffled":  # adversarial order: the full-sort (slow) path
        paths = shuffle_rows(paths, tmp_path / "shuf", 5, seed=3)
    shards = _shards(paths)
    if variant == "dups_filters":  # out-of-grid and over-ceiling rows
        shards.append(HEADER + b"\nj000001,2021-05-09 12:00:00,45.0,-92.0,65101,10,10\n"
                      b"j000002,2021-05-09 12:00:01,37.0,-92.0,65101,300,10\n")
    spec = cvlg.GridSpec()
    st = cvlg.PipelineStats()
    lat, feats = cvlg.journey_features_host(shards, spec, stop_speed=20.0, stats=st)
    # the lattice is unchanged by the feature request
    plain = cvlg.run_pipeline_host(shards, spec)
    assert np.array_equal(plain.planes, lat.planes)
    kept = fo.kept_records(ref, shards, spec, hp=hp)
    rows = fo.features_table(kept, 20.0)
    _compare(rows, feats, cvlg.journey_ids(shards, feats))
    assert sum(int(x) for x in feats["points"]) == st.accepted
    mn, mx = fo.cell_extremes(kept, spec.dims())
    assert np.array_equal(feats["cell_speed_min"].view(np.uint32), mn.view(np.uint32))
    assert np.array_equal(feats["cell_speed_max"].view(np.uint32), mx.view(np.uint32))
