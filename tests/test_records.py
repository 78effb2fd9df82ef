"""The secondary boundary cvl::run_pipeline_from_records (aggregate.hpp:130-133): already-parsed
records with provenance through cvlg_run_pipeline_records against the UNMODIFIED reference
function on the same records. Lattice bits, raw counts and statistics must be identical."""
from __future__ import annotations

import datetime
import random

import pytest

from helpers import diff_lattice, stats_dict

pytestmark = pytest.mark.gpu


def _epoch(text: bytes) -> int:
    d = datetime.datetime.strptime(text.decode(), "%Y-%m-%d %H:%M:%S")
    return int((d - datetime.datetime(1970, 1, 1)).total_seconds())


def _records_of_day(seed, journeys, shards, mean_duration=300.0):
    import paper_2305_07454_b200 as cvlg
    blob, offs, _ = cvlg.synth_day(seed=seed, journeys=journeys, shards=shards,
                                   mean_duration=mean_duration)
    recs = []
    for s in range(shards):
        lines = blob[offs[s]:offs[s + 1]].tobytes().split(b"\n")[1:]
        path = b"/data/day/shard_%04d.csv" % s
        for ln, line in enumerate(lines, start=1):
            if not line:
                continue
            f = line.split(b",")
            recs.append((f[0], _epoch(f[1]), float(f[2]), float(f[3]), f[4], float(f[5]),
                         float(f[6]), path, ln))
    return recs


def _check(ref, recs, spec, rules=None):
    import paper_2305_07454_b200 as cvlg
    ep, er, est = ref.run_pipeline_from_records(recs, spec, rules, n_partitions=4, n_threads=4)
    st = cvlg.PipelineStats()
    lat = cvlg.run_pipeline_from_records(recs, spec, rules, n_partitions=3, stats=st)
    d = diff_lattice(ep, er, lat.planes, lat.raw)
    assert d == "", d
    assert stats_dict(st) == est
    return est


def test_records_synth_day_any_order(ref):
    """A synthetic day's parsed rows, handed over in a random order (the provenance sort must
    restore the reference's (path rank, line) order), default and fine grids."""
    import paper_2305_07454_b200 as cvlg
    recs = _records_of_day(seed=4, journeys=300, shards=3)
    random.Random(1).shuffle(recs)
    est = _check(ref, recs, cvlg.GridSpec())
    assert est["rows_read"] == len(recs) and est["parsed"] == len(recs)
    _check(ref, recs, cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1))


def test_records_duplicates_conflicts_and_edges(ref):
    """Duplicate (journey, time) pairs across paths (the min-provenance survivor; equal and
    conflicting payloads), values no parser would let through (heading 360, latitudes off the
    grid and out of range, speeds over the ceiling, an infinite speed), empty and long journey ids,
    line numbers past 2^32 (the reference keeps the low 32 bits)."""
    import paper_2305_07454_b200 as cvlg
    base = _records_of_day(seed=6, journeys=120, shards=2)
    rng = random.Random(3)
    recs = list(base)
    for r in rng.sample(base, 400):  # duplicates: same key, other path; half conflicting
        jid, ts, la, lo, pc, sp, hd, path, ln = r
        other = b"/data/day/a_first.csv" if rng.random() < 0.5 else b"/data/day/z_last.csv"
        if rng.random() < 0.5:
            sp = sp + 1.0
        recs.append((jid, ts, la, lo, pc, sp, hd, other, rng.randrange(1, 10_000)))
    edges = [
        (b"edge-heading", 1_620_600_000, 38.0, -92.0, b"65101", 30.0, 360.0, b"/e.csv", 1),
        (b"edge-heading", 1_620_600_001, 38.0, -92.0, b"65101", 30.0, 359.9999999, b"/e.csv", 2),
        (b"edge-offgrid", 1_620_600_000, 45.0, -92.0, b"", 30.0, 10.0, b"/e.csv", 3),
        (b"edge-range", 1_620_600_000, 95.0, -92.0, b"", 30.0, 10.0, b"/e.csv", 4),
        (b"edge-speed", 1_620_600_000, 38.0, -92.0, b"", 300.0, 10.0, b"/e.csv", 5),
        (b"edge-inf", 1_620_600_000, 38.0, -92.0, b"", float("inf"), 10.0, b"/e.csv", 6),
        (b"", 1_620_600_000, 38.0, -92.0, b"", 30.0, 10.0, b"/e.csv", 7),
        (b"a-journey-id-longer-than-fifteen", 1_620_600_000, 37.0, -91.0, b"x", 20.0, 90.0,
         b"/e.csv", (1 << 32) + 8),
        (b"a-journey-id-longer-than-fifteen", 1_620_600_003, 37.01, -91.0, b"x", 21.0, 90.0,
         b"/e.csv", 9),
        (b"edge-neg", -86_399, 38.0, -92.0, b"", 30.0, 10.0, b"/e.csv", 10),
    ]
    recs += edges
    rng.shuffle(recs)
    est = _check(ref, recs, cvlg.GridSpec())
    assert est["duplicates_dropped"] == 400 and est["conflicting_duplicates"] > 0
    assert sum(est["filtered"].values()) > 0
    _check(ref, recs, cvlg.GridSpec(lat_step=0.25, lon_step=0.25))


def test_records_errors_and_empty(ref):
    """ZeroPartitions and OutOfBounds (require_in_grid = false with an off-grid record) like
    the reference; an empty record set gives the empty lattice."""
    import paper_2305_07454_b200 as cvlg
    from oracle.oracle import RefError
    recs = _records_of_day(seed=2, journeys=20, shards=1)
    with pytest.raises(cvlg.CvlError):
        cvlg.run_pipeline_from_records(recs, cvlg.GridSpec(), n_partitions=0)
    off = recs + [(b"x", 1_620_600_000, 45.0, -92.0, b"", 30.0, 10.0, b"/o.csv", 1)]
    rules = cvlg.FilterRules(require_in_grid=False)
    with pytest.raises(RefError):
        ref.run_pipeline_from_records(off, cvlg.GridSpec(), rules)
    with pytest.raises(cvlg.CvlError):
        cvlg.run_pipeline_from_records(off, cvlg.GridSpec(), rules)
    _check(ref, [], cvlg.GridSpec())
