"""Shared test helpers: input builders and the frame comparator (compare_days analogue,
proj/tests/acceptance.cpp:99-120, here bit-exact)."""
from __future__ import annotations

import random
from pathlib import Path

import numpy as np

HEADER = b"Journey Id,Timestamp,Latitude,Longitude,Postal Code,Speed,Heading"


def write_shards(dirpath: Path, contents: list[bytes], prefix="shard_") -> list[str]:
    dirpath.mkdir(parents=True, exist_ok=True)
    paths = []
    for i, c in enumerate(contents):
        p = dirpath / f"{prefix}{i:04d}.csv"
        p.write_bytes(c)
        paths.append(str(p))
    return paths


def shuffle_rows(paths: list[str], out_dir: Path, n_out: int, seed: int) -> list[str]:
    """Adversarial variant: all data rows shuffled across n_out shards."""
    rows = []
    for p in paths:
        lines = Path(p).read_bytes().split(b"\n")
        rows.extend(l for l in lines[1:] if l)
    rng = random.Random(seed)
    rng.shuffle(rows)
    contents = [HEADER + b"\n" + b"\n".join(rows[i::n_out]) + b"\n" for i in range(n_out)]
    return write_shards(out_dir, contents)


def diff_lattice(exp_planes, exp_raw, got_planes, got_raw) -> str:
    """'' when bit-identical, else a description of the first divergence."""
    if exp_planes.shape != got_planes.shape:
        return f"shape {exp_planes.shape} vs {got_planes.shape}"
    for ch in range(8):
        a, b = exp_planes[:, ch], got_planes[:, ch]
        if not np.array_equal(a, b):
            idx = np.argwhere(a != b)[0]
            what = "speed" if ch < 4 else "volume"
            return (f"{what} d={ch % 4} differs at t={idx[0]} r={idx[1]} c={idx[2]}: "
                    f"{a[tuple(idx)]:#x} vs {b[tuple(idx)]:#x} "
                    f"({int((a != b).sum())} cells differ)")
    if exp_raw is not None and got_raw is not None and not np.array_equal(exp_raw, got_raw):
        idx = np.argwhere(exp_raw != got_raw)[0]
        return f"raw_count differs at {tuple(idx)}: {exp_raw[tuple(idx)]} vs {got_raw[tuple(idx)]}"
    return ""


def stats_dict(st) -> dict:
    return {
        "rows_read": st.rows_read, "parsed": st.parsed,
        "duplicates_dropped": st.duplicates_dropped,
        "conflicting_duplicates": st.conflicting_duplicates, "accepted": st.accepted,
        "rejected": dict(st.rejected), "filtered": dict(st.filtered),
    }


def commuter_days(n_journeys, days, cells, seed):
    """Every journey drives in the same 10 minutes of every day, hopping among `cells` nearby
    0.01-degree cells with random headings: each day reopens the time bins of the previous days
    (the fold's time-bin-window reload path); > 10 cells per window overflows the lane table."""
    rng = random.Random(seed)
    hmax = 80.0 if cells <= 8 else 360.0  # one heading sector: <= cells codes per window
    out = []
    for d in range(days):
        lines = []
        for j in range(n_journeys):
            base_lat = 37.0 + (j % 40) * 0.05
            base_lon = -93.0 + (j // 40) * 0.05
            pts = [(base_lat + 0.01 * (k % 4) + 0.003, base_lon + 0.01 * (k // 4) + 0.004)
                   for k in range(cells)]
            for sec in range(0, 600, 3 + j % 3):
                la, lo = pts[rng.randrange(cells)]
                lines.append(b"c%05d,2021-05-%02d 08:%02d:%02d,%.6f,%.6f,65101,%.2f,%.2f" % (
                    j, 9 + d, sec // 60, sec % 60, la, lo, rng.uniform(0, 80), rng.uniform(0, hmax)))
        out.append(HEADER + b"\n" + b"\n".join(lines) + b"\n")
    return out


def malformed_contents(seed: int = 5) -> list[bytes]:
    """Shards exercising read_shard / parse_record_impl edge cases (ingest.cpp:119-157, 195-239):
    CRLF, blank lines, no trailing newline, an empty shard, a BadHeader shard, a permuted header,
    a header-only shard, plus the malformed-line corpus mixed with good lines."""
    import corpus
    rng = random.Random(seed)
    body = corpus.line_corpus(rng, 3000)
    good = [b"jj%03d,2021-05-09 %02d:%02d:%02d,%.6f,%.6f,65101,%.2f,%.2f" % (
        i % 17, (i // 3600) % 24, (i // 60) % 60, i % 60, 36.1 + (i % 400) * 0.01,
        -95.7 + (i % 600) * 0.011, (i * 7.3) % 140, (i * 13.7) % 360) for i in range(4000)]
    mixed = body + good
    rng.shuffle(mixed)
    return [
        HEADER + b"\r\n" + b"\r\n".join(mixed[:1500]) + b"\r\n",
        HEADER + b"\n" + b"\n\n".join(mixed[1500:4000]),  # blank lines, no trailing newline
        b"",  # empty shard: no header, no rows
        b"nope,nope\n1,2\n",  # BadHeader
        b"heading,speed,zip code,longitude,latitude,timestamp,journey-id\n" + b"\n".join(
            b"%s,%s,%s,%s,%s,%s,%s" % tuple(reversed(l.split(b",")[:7])) for l in good[:800]
            if len(l.split(b",")) == 7),
        HEADER,  # header only, no newline
        HEADER + b"\n" + b"\n".join(mixed[4000:]) + b"\n",
    ]
