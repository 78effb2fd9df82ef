"""TEST INFRASTRUCTURE: CPU restatement of the per-journey feature table
(paper_2305_07454_b200/csrc/features.cu). The reference has no such function:
parity for these columns is UNPINNED against the reference and pinned only against this file,
whose record selection reuses the reference's own parser (oracle/_ref: parse_record_impl,
ingest.cpp:119-157) and the repo's reference-pinned binning restatement (grid.cuh via
tests/native/hostparse.cpp), and whose formulas are checked on hand-computed traces
(tests/test_features.py::test_restatement_known_answers).

Record set = the records the lattice aggregates: accepted lines, first of each (journey, epoch)
group in provenance order (aggregate.cpp:266-291), passing filter_reason (aggregate.cpp:48-56).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

EARTH_R = 6371008.8
DEG = 0.017453292519943295


def haversine_m(la1, lo1, la2, lo2):
    p1, p2 = la1 * DEG, la2 * DEG
    dp, dl = (la2 - la1) * DEG, (lo2 - lo1) * DEG
    s1, s2 = math.sin(0.5 * dp), math.sin(0.5 * dl)
    a = s1 * s1 + math.cos(p1) * math.cos(p2) * s2 * s2
    return 2.0 * EARTH_R * math.asin(math.sqrt(min(1.0, a)))


def journey_features(records, stop_speed):
    """records: list of (epoch, lat, lon, speed) of ONE journey in timestamp order."""
    f = dict(points=0, t_first=0, t_last=0, length_m=0.0, max_step_m=0.0, max_speed=0.0,
             max_abs_accel=0.0, dwell_s=0.0, stops=0)
    prev = None
    for t, la, lo, sp in records:
        stopped = sp <= stop_speed
        if prev is None:
            f["t_first"] = t
            if stopped:
                f["stops"] += 1
        else:
            pt, pla, plo, psp, pst = prev
            dt = float(t - pt)
            step = haversine_m(pla, plo, la, lo)
            f["length_m"] += step
            f["max_step_m"] = max(f["max_step_m"], step)
            f["max_abs_accel"] = max(f["max_abs_accel"], abs(sp - psp) / dt)
            if stopped and pst:
                f["dwell_s"] += dt
            if stopped and not pst:
                f["stops"] += 1
        f["max_speed"] = max(f["max_speed"], sp)
        f["points"] += 1
        f["t_last"] = t
        prev = (t, la, lo, sp, stopped)
    return f


def kept_records(ref, shards, spec, rules=None, hp=None):
    """(id bytes, epoch, lat, lon, speed, cell code or None) of the aggregated records, from
    shard byte strings in rank order."""
    rules = rules or {"require_in_grid": True, "speed_ceiling": 250.0}
    g = spec.__dict__ if hasattr(spec, "__dict__") else spec
    seen = {}
    for si, blob in enumerate(shards):
        lines = blob.split(b"\n")
        if not lines or not lines[0].rstrip(b"\r"):
            continue
        cols = ref.parse_header(lines[0].rstrip(b"\r") if lines[0].endswith(b"\r") else lines[0])
        if cols is None:
            continue
        for li, raw in enumerate(lines[1:], start=2):
            line = raw[:-1] if raw.endswith(b"\r") else raw
            if not line:
                continue
            why, rec = ref.parse_record(line, cols)
            if why != -1:
                continue
            key = (rec.journey_id, rec.epoch_sec)
            if key in seen:
                continue  # duplicate: the min-provenance survivor came first
            seen[key] = (rec.journey_id, rec.epoch_sec, rec.latitude, rec.longitude, rec.speed,
                         rec.heading)
    out = []
    for jid, t, la, lo, sp, hd in seen.values():
        in_grid = g["lat_min"] <= la <= g["lat_max"] and g["lon_min"] <= lo <= g["lon_max"]
        if rules["require_in_grid"] and not in_grid:
            continue
        if sp > rules["speed_ceiling"]:
            continue
        code = None
        if hp is not None and in_grid:
            gd = (ctypes.c_double * 7)(g["lat_min"], g["lat_max"], g["lon_min"], g["lon_max"],
                                       g["lat_step"], g["lon_step"], g["dxn_offset"])
            gi = (ctypes.c_uint32 * 2)(g["min_step"], g["dxn_step"])
            code = hp.hp_cell_code(gd, gi, 1, rules["speed_ceiling"], t, la, lo, sp, hd)
        out.append((jid, t, la, lo, sp, code))
    return out


def features_table(kept, stop_speed):
    by = {}
    for jid, t, la, lo, sp, _ in kept:
        by.setdefault(jid, []).append((t, la, lo, sp))
    rows = []
    for jid in sorted(by):  # lexicographic id order = the lattice's journey rank order
        rows.append((jid, journey_features(sorted(by[jid]), stop_speed)))
    return rows


def cell_extremes(kept, dims):
    T, D, R, C = dims
    mn = np.zeros((T, 4, R, C), dtype=np.float32)
    mx = np.zeros((T, 4, R, C), dtype=np.float32)
    seen = np.zeros((T, 4, R, C), dtype=bool)
    for _, _, _, _, sp, code in kept:
        t, rem = divmod(code, D * R * C)
        d, rc = divmod(rem, R * C)
        r, c = divmod(rc, C)
        v = np.float32(sp)
        if not seen[t, d, r, c]:
            mn[t, d, r, c] = mx[t, d, r, c] = v
            seen[t, d, r, c] = True
        else:
            mn[t, d, r, c] = min(mn[t, d, r, c], v)
            mx[t, d, r, c] = max(mx[t, d, r, c], v)
    return mn, mx
