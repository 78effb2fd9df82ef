"""TEST CODE: a plain-Python restatement of the multi-GPU line routing (csrc/route.cu), used as
the checker of the routing kernels and of the exchange layout.

The reference routes every parsed record to journey_hash(journey_id) % P
(proj/src/aggregate.cpp:432-438; journey_hash = FNV-1a 64, ingest.cpp:287-291). A record's
journey_id is the trimmed journey_id field of its line (split_fields / trim, ingest.cpp:31-53)
after read_shard stripped one trailing '\\r' (ingest.cpp:203-210); empty lines are not rows
(ingest.cpp:227). The hash here is the reference's own (oracle/_ref ref_journey_hash) when a
`ref` is given, else a Python FNV-1a.
"""
from __future__ import annotations

from pathlib import Path


def fnv1a(b: bytes) -> int:
    h = 1469598103934665603
    for c in b:
        h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def line_owner(raw: bytes, id_col: int, n: int, hash_fn=fnv1a):
    """Owner of one line (without its '\\n'); None for lines that are not rows."""
    if raw == b"" or raw == b"\r":
        return None
    content = raw[:-1] if raw.endswith(b"\r") else raw
    fields = content.split(b",")
    f = fields[id_col] if 0 <= id_col < len(fields) else b""
    return hash_fn(f.strip(b" \t\r")) % n


def header_of(path: str) -> tuple[bytes, int]:
    """(header line incl. '\\n', first data byte)."""
    data = Path(path).read_bytes()
    nl = data.find(b"\n")
    if nl < 0:
        return data + b"\n", len(data)
    return data[: nl + 1], nl + 1


def streams(paths_ranked: list[str], pieces: list[tuple[int, int, int]], id_cols: list[int], n: int,
            hash_fn=fnv1a):
    """Per owner: the stream bytes this part sends (per piece: header, then its lines routed
    there, each ending in '\\n') and the offset of each piece's header in it."""
    out = [bytearray() for _ in range(n)]
    vs = [[] for _ in range(n)]
    for file, off, ln in pieces:
        hdr, _ = header_of(paths_ranked[file])
        data = Path(paths_ranked[file]).read_bytes()[off: off + ln]
        lines = data.split(b"\n")
        if data.endswith(b"\n"):
            lines = lines[:-1]
        for o in range(n):
            vs[o].append(len(out[o]))
            out[o] += hdr
        for raw in lines:
            o = line_owner(raw, id_cols[file], n, hash_fn)
            if o is not None:
                out[o] += raw + b"\n"
    return [bytes(b) for b in out], vs
