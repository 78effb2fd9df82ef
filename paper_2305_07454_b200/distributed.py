"""Multi-GPU pipeline: one process per GPU, journeys sharded by FNV-1a id hash.

The reference partitions work by `journey_hash(id) % P` (proj/src/ingest.cpp:287-301,
aggregate.cpp:433-438) and journeys never straddle partitions (aggregate.cpp:372-373). Here the
partitions are GPUs: every rank decodes / dedups / orders / folds ITS journeys on its own
device (no communication), producing per-(cell, journey) subtotals. The only exchange is the
per-cell combine, which must fold subtotals in GLOBAL journey order to stay bit-exact:

  1. each rank exports (cell, journey key, f64 sum, count) tuples with exact global keys;
  2. tuples go to the rank owning the cell's time slab (NCCL all-to-all over NVLink);
  3. each rank folds its slab (cvlg_finalize_pairs: (cell, key) order = the reference's
     finalize, aggregate.cpp:161-204) into a lattice that is zero outside the slab;
  4. one NCCL all-reduce (SUM over u32 words; slabs are disjoint, so this is a bitwise union)
     leaves the full lattice on every rank.

`slab_owner` and `exchange_tuples` are device-agnostic torch code (tested with gloo on CPU in
tests/test_distributed.py); the fold itself is the sm_100a library.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import cvlg as _c

_lib = _c.lib()
_vp = ctypes.c_void_p
_lib.cvlg_partial_device.argtypes = [_vp, _vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t,
                                     ctypes.POINTER(_c._Grid), ctypes.POINTER(_c._Rules),
                                     ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(_c._Stats),
                                     _vp]
_lib.cvlg_export_pairs.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.cvlg_finalize_pairs.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_uint64,
                                     ctypes.POINTER(_c._Grid), _vp, _vp, _vp]
_lib.cvlg_synth_day_owned.restype = ctypes.c_int64
_lib.cvlg_synth_day_owned.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_int32, _vp,
                                      ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _vp,
                                      ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.POINTER(ctypes.c_uint64)]

STAT_KEYS = ["rows_read", "parsed", "duplicates_dropped", "conflicting_duplicates", "accepted"]


def synth_day_owned(seed: int, journeys: int, shards: int, mean_duration: float, mod: int,
                    rem: int, sample_period: float = 1.0, day: str = "2021-05-09"):
    """The share of a `journeys`-journey synthetic day owned by rank `rem` of `mod`."""
    import datetime

    import numpy as np
    d = datetime.date.fromisoformat(day)
    day_number = (d - datetime.date(1970, 1, 1)).days
    max_rows = (journeys // max(mod, 1) + 64 + journeys // 20) * (int(1.7 * mean_duration / sample_period) + 2)
    cap = max_rows * 80 + shards * 80 + 64
    out = np.empty(cap, dtype=np.uint8)
    offs = (ctypes.c_uint64 * (shards + 1))()
    rows = ctypes.c_uint64()
    n = _lib.cvlg_synth_day_owned(seed, journeys, shards, sample_period, mean_duration, day_number,
                                  None, 0, mod, rem, out.ctypes.data_as(_vp), cap, offs,
                                  ctypes.byref(rows))
    if n < 0:
        raise _c.CvlError(101, f"synth_day_owned failed ({n})")
    return out[:n], list(offs), rows.value


def slab_owner(cell: torch.Tensor, cells_per_t: int, n_batches: int, world: int) -> torch.Tensor:
    """Rank owning each cell: contiguous time slabs, rank r owns t in [r*T/W, (r+1)*T/W)."""
    t = torch.div(cell, cells_per_t, rounding_mode="floor")
    return torch.div(t * world, n_batches, rounding_mode="floor")


def exchange_tuples(cols: torch.Tensor, owner: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-to-all of int64 tuple rows (n, k) so that every row reaches its owner rank."""
    order = torch.argsort(owner, stable=True)
    send = cols.index_select(0, order).contiguous()
    counts = torch.bincount(owner, minlength=world).to(torch.int64)
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts, group=group)
    in_splits = counts.tolist()
    out_splits = recv_counts.tolist()
    recv = torch.empty((int(sum(out_splits)), cols.shape[1]), dtype=cols.dtype, device=cols.device)
    dist.all_to_all_single(recv, send, out_splits, in_splits, group=group)
    return recv


def run_pipeline_distributed(d_csv: torch.Tensor, shard_offsets, spec: _c.GridSpec | None = None,
                             rules: _c.FilterRules | None = None, ctx: _c.Context | None = None,
                             group=None, stats: dict | None = None):
    """This rank's CSV (its journeys) in HBM -> the full lattice on every rank.
    Returns (planes [T,8,R,C] int32 view of u32, raw [T,4,R,C])."""
    spec = spec or _c.GridSpec()
    rules = rules or _c.FilterRules()
    ctx = ctx or _c.default_context()
    world = dist.get_world_size(group)
    dev = d_csv.device
    stream = torch.cuda.current_stream(dev).cuda_stream
    T, D, R, C = spec.dims()
    offs = (ctypes.c_uint64 * len(shard_offsets))(*shard_offsets)
    n = ctypes.c_uint64()
    st = _c._Stats()
    _c._check(_lib.cvlg_partial_device(ctx.handle, _vp(d_csv.data_ptr()), offs,
                                       len(shard_offsets) - 1, ctypes.byref(spec._c()),
                                       ctypes.byref(rules._c()), ctypes.byref(n), ctypes.byref(st),
                                       _vp(stream) if stream else None))
    n = n.value
    cols = torch.empty((max(n, 1), 5), dtype=torch.int64, device=dev)
    # export straight into strided columns: write to contiguous column buffers, then stack
    cell = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    k0 = torch.empty_like(cell)
    k1 = torch.empty_like(cell)
    s = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    cnt = torch.empty_like(cell)
    _c._check(_lib.cvlg_export_pairs(ctx.handle, _vp(cell.data_ptr()), _vp(k0.data_ptr()),
                                     _vp(k1.data_ptr()), _vp(s.data_ptr()), _vp(cnt.data_ptr()),
                                     _vp(stream) if stream else None))
    cols = torch.stack([cell, k0, k1, s.view(torch.int64), cnt], dim=1)[:n]
    owner = slab_owner(cols[:, 0], D * R * C, T, world)
    recv = exchange_tuples(cols, owner, world, group)
    m = recv.shape[0]
    rc = [recv[:, i].contiguous() for i in range(5)]
    planes = torch.empty((T, 8, R, C), dtype=torch.int32, device=dev)
    raw = torch.empty((T, 4, R, C), dtype=torch.int32, device=dev)
    _c._check(_lib.cvlg_finalize_pairs(ctx.handle, _vp(rc[0].data_ptr()), _vp(rc[1].data_ptr()),
                                       _vp(rc[2].data_ptr()), _vp(rc[3].data_ptr()),
                                       _vp(rc[4].data_ptr()), m, ctypes.byref(spec._c()),
                                       _vp(planes.data_ptr()), _vp(raw.data_ptr()),
                                       _vp(stream) if stream else None))
    dist.all_reduce(planes, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(raw, op=dist.ReduceOp.SUM, group=group)
    if stats is not None:
        vals = [st.rows_read, st.parsed, st.duplicates_dropped, st.conflicting_duplicates,
                st.accepted, *st.rejected, *st.filtered]
        t = torch.tensor(vals, dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        v = t.tolist()
        stats.clear()
        stats.update(dict(zip(STAT_KEYS, v[:5])))
        stats["rejected"] = {k: x for k, x in zip(_c.REJECT_NAMES, v[5:10]) if x}
        stats["filtered"] = dict(zip(_c.FILTER_NAMES, v[10:13]))
    return planes, raw
