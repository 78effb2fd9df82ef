#!/usr/bin/env python
"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference library
(oracle/_ref, compiled from /root/reference/proj/src). Run in the build container:

    python tests/golden/make_golden.py

Outputs (committed; the GPU box has no /root/reference):
  parse_kat.json     data lines -> reference ParseReason / field f64 bit patterns
  numeric_kat.json   numeric fields -> parse_double accept/reject + f64 bits
  header_kat.json    header lines -> ColumnMap
  grid_kat.json      (grid, value) -> lat/lon/time/dxn bins or OutOfBounds, grid dims
  days/<case>/       small shard sets (CSV) + expected.npz (planes, raw) + expected.json (stats,
                     container sha256)
"""
from __future__ import annotations

import hashlib
import json
import random
import struct
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.oracle import Ref  # noqa: E402
import corpus  # noqa: E402
from helpers import HEADER, shuffle_rows, write_shards  # noqa: E402


class Spec:
    def __init__(self, **kw):
        d = dict(lat_min=36.0, lat_max=40.6, lon_min=-95.8, lon_max=-89.1, lat_step=0.1,
                 lon_step=0.1, min_step=5, dxn_step=90, dxn_offset=0.0)
        d.update(kw)
        self.__dict__.update(d)

    def as_dict(self):
        return dict(self.__dict__)


class Rules:
    def __init__(self, require_in_grid=True, speed_ceiling=250.0, drop_missing=True):
        self.require_in_grid = require_in_grid
        self.speed_ceiling = speed_ceiling
        self.drop_missing = drop_missing


def bits(x: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", x))[0]


CANON = [0, 1, 2, 3, 4, 5, 6, 7]


def gen_parse(ref: Ref):
    rng = random.Random(20230512)
    lines = corpus.line_corpus(rng, 1500)
    out = []
    for ln in lines:
        why, rec = ref.parse_record(ln, CANON)
        e = {"line": ln.decode("latin-1"), "reason": why}
        if why == -1:
            e.update(epoch=rec.epoch_sec, lat=bits(rec.latitude), lon=bits(rec.longitude),
                     speed=bits(rec.speed), heading=bits(rec.heading),
                     id=rec.journey_id.decode("latin-1"), postal=rec.postal_code.decode("latin-1"))
        out.append(e)
    (HERE / "parse_kat.json").write_text(json.dumps(out, indent=0))

    nums = corpus.numeric_corpus(random.Random(7), 6000)
    nout = []
    for s in nums:
        v = ref.from_chars(s.encode("utf-8"))
        nout.append({"s": s, "bits": None if v is None else bits(v)})
    (HERE / "numeric_kat.json").write_text(json.dumps(nout, indent=0))

    hout = []
    for h in corpus.HEADER_CORPUS:
        hout.append({"header": h.decode("latin-1"), "cols": ref.parse_header(h)})
    (HERE / "header_kat.json").write_text(json.dumps(hout, indent=0))

    ts = []
    for t in corpus.TIMESTAMP_EDGE:
        ts.append({"ts": t, "epoch": ref.timestamp(t.encode())})
    (HERE / "timestamp_kat.json").write_text(json.dumps(ts, indent=0))


def gen_grid(ref: Ref):
    rng = random.Random(99)
    grids = [Spec(), Spec(lat_step=0.25, lon_step=0.25), Spec(lat_step=10, lon_step=10),
             Spec(lat_min=36.0, lat_max=36.1, lon_min=-93.0, lon_max=-92.8, lat_step=0.01,
                  lon_step=0.01),
             Spec(lat_min=36.0, lat_max=38.0, lon_min=-93.0, lon_max=-92.0, lat_step=0.01,
                  lon_step=0.01),
             Spec(dxn_offset=45.0), Spec(min_step=60), Spec(dxn_step=120, dxn_offset=-30.0),
             Spec(lat_min=-100.0, lat_max=-100.0 + 300 * 0.013, lat_step=0.013),
             Spec(lat_min=-100.0, lat_max=-100.0 + 300 * 0.007, lat_step=0.007, lon_step=0.007)]
    out = []
    for g in grids:
        e = {"grid": g.as_dict(), "rows": ref.bin(g, 4)[1], "cols": ref.bin(g, 5)[1], "cases": []}
        vals = []
        for k in range(0, 310, 7):
            vals.append(g.lat_min + k * g.lat_step)  # f64-computed bin edges (test_grid.cpp:143)
        for _ in range(150):
            vals.append(rng.uniform(g.lat_min - 0.5, g.lat_max + 0.5))
        vals += [g.lat_min, g.lat_max, 37.664087, 36.05]
        for v in vals:
            e["cases"].append(["lat", bits(v), *ref.bin(g, 0, v)])
        for _ in range(150):
            v = rng.uniform(g.lon_min - 0.5, g.lon_max + 0.5)
            e["cases"].append(["lon", bits(v), *ref.bin(g, 1, v)])
        for v in [0.0, 33.0, 90.0, 359.9, 269.999, 350.0, 46.0, 180.0, 270.0, 359.9999999,
                  359.99999964, 44.99999999999] + [rng.uniform(0, 360) for _ in range(100)]:
            e["cases"].append(["dxn", bits(v), *ref.bin(g, 3, v)])
        for ep in [0, 1620531522, -1, -86400, 1620604799, 1620518400 + 45 * 300] + \
                  [rng.randrange(-10 ** 10, 10 ** 10) for _ in range(60)]:
            e["cases"].append(["time", ep, *ref.bin(g, 2, 0.0, ep)])
        out.append(e)
    (HERE / "grid_kat.json").write_text(json.dumps(out, indent=0))


def save_day(ref: Ref, name: str, paths: list[str], spec: Spec, rules: Rules | None = None):
    d = HERE / "days" / name
    planes, raw, st, _ = ref.run_pipeline(paths, spec, rules)
    with tempfile.TemporaryDirectory() as t:
        cpath = Path(t) / "x.cvl1"
        ref.write_container(planes, spec, 18756, cpath)
        sha = hashlib.sha256(cpath.read_bytes()).hexdigest()
    np.savez_compressed(d / "expected.npz", planes=planes, raw=raw)
    meta = {"grid": spec.as_dict(), "stats": st, "container_sha256_day18756": sha,
            "rules": None if rules is None else rules.__dict__,
            "shards": [Path(p).name for p in paths]}
    (d / "expected.json").write_text(json.dumps(meta, indent=1))


def gen_days(ref: Ref):
    base = HERE / "days"
    with tempfile.TemporaryDirectory() as t:
        t = Path(t)
        # 1. small synthetic day (reference generator), coarse grid
        ref.generate_day(t / "a", seed=1, journeys=24, shards=3, mean_duration=150.0)
        src = sorted(str(p) for p in (t / "a").glob("*.csv"))
        paths = write_shards(base / "synth_small", [Path(p).read_bytes() for p in src])
        save_day(ref, "synth_small", paths, Spec(lat_step=0.25, lon_step=0.25))
        # 2. duplicates (sample_period 0.5), degenerate 1x1 grid
        ref.generate_day(t / "b", seed=5, journeys=10, shards=2, sample_period=0.5,
                         mean_duration=60.0)
        src = sorted(str(p) for p in (t / "b").glob("*.csv"))
        sh = shuffle_rows(src, t / "bs", 3, seed=2)
        paths = write_shards(base / "dups_shuffled", [Path(p).read_bytes() for p in sh])
        save_day(ref, "dups_shuffled", paths, Spec(lat_step=10.0, lon_step=10.0))
        # 3. malformed lines, CRLF, blank lines, BadHeader shard, empty shard, permuted header
        rng = random.Random(3)
        body = corpus.line_corpus(rng, 200)
        good = [b"jj%03d,2021-05-09 %02d:%02d:%02d,%.6f,%.6f,65101,%.2f,%.2f" % (
            i % 7, (i // 3600) % 24, (i // 60) % 60, i % 60, 36.1 + (i % 40) * 0.1,
            -95.7 + (i % 60) * 0.11, (i * 7.3) % 140, (i * 13.7) % 360) for i in range(600)]
        mixed = body + good
        rng.shuffle(mixed)
        contents = [
            HEADER + b"\r\n" + b"\r\n".join(mixed[:300]) + b"\r\n",
            HEADER + b"\n" + b"\n\n".join(mixed[300:600]),
            b"",
            b"nope,nope\n1,2\n",
            b"heading,speed,zip code,longitude,latitude,timestamp,journey-id\n" + b"\n".join(
                b",".join(reversed(l.split(b",")[:7])) for l in good[:100]),
            HEADER + b"\n" + b"\n".join(mixed[600:]) + b"\n",
        ]
        paths = write_shards(base / "malformed", contents)
        save_day(ref, "malformed", paths, Spec(lat_step=0.5, lon_step=0.5, min_step=60))
        # 4. Table-1 snapshot rows (acceptance.cpp:248-253)
        rows = [b"33456rd,2021-05-09 03:48:42,37.664087,-92.6546,65536,105.98,33",
                b"31224tf,2021-05-09 03:49:42,37.667707,-92.6490,65536,0,53",
                b"22124fs,2021-05-09 03:49:49,37.690978,-92.6490,65536,48.38,33",
                b"33456rd,2021-05-09 03:48:42,37.664087,-92.6546,65536,105.98,33"]
        paths = write_shards(base / "table1", [HEADER + b"\n" + b"\n".join(rows) + b"\n"])
        save_day(ref, "table1", paths, Spec(lat_step=10.0, lon_step=10.0))


def main():
    ref = Ref()
    gen_parse(ref)
    gen_grid(ref)
    gen_days(ref)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
