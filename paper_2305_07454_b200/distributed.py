"""Multi-GPU pipeline for one process per GPU (torchrun), journeys sharded by FNV-1a id hash.

The reference partitions records by `journey_hash(id) % P` (proj/src/ingest.cpp:287-291,
aggregate.cpp:414-443); journeys never straddle partitions (aggregate.cpp:372-373) and the merged
entries are finalized in (cell, journey id) order (aggregate.cpp:161-204). Here the partitions
are ranks. Every step that touches data is an sm_100a kernel of the C ABI (include/cvlg.h,
csrc/route.cu + multi.cu); torch.distributed only moves bytes:

  1. cvlg_route_stage    rank r streams its 1/N byte range of the shards (cut at line
                         boundaries) into HBM and counts, per owner, the bytes of the lines
                         whose journey hashes there;
  2. cvlg_route_scatter  writes every line (and each piece's header line) into a send buffer
                         partitioned by owner; one all-to-all (NCCL) delivers the streams, which
                         the owner concatenates in source order = the reference's provenance
                         order (shard rank, line);
  3. cvlg_partial_device the owner's journeys through the single-GPU pipeline, up to the
                         per-(cell, journey) subtotals;
  4. cvlg_tuples_*       subtotals as (cell, exact journey key, f64 sum, count) tuples,
                         partitioned by the cell's time-slab owner; one all-to-all;
  5. cvlg_finalize_tuples each rank folds its slab; slabs are all-gathered (the lattice rows are
                         disjoint, so no reduction is needed).

The single-process twin (one host thread, peer stores instead of all-to-alls) is
cvlg_run_pipeline_multi / cvlg.MultiGPU. The byte-layout arithmetic below (stream_layout,
virtual_shards) is plain Python so it is tested on CPU with gloo (tests/test_distributed.py).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import cvlg as _c

_lib = _c.lib()
_vp = ctypes.c_void_p
TUPLE_BYTES = 40  # (u64 cell, u64 key0, u64 key1, f64 sum, u64 count)
STAT_KEYS = ["rows_read", "parsed", "duplicates_dropped", "conflicting_duplicates", "accepted"]

# the old synthetic helper (pre-sharded generator output) is kept for tests of the combine
_lib.cvlg_synth_day_owned.restype = ctypes.c_int64
_lib.cvlg_synth_day_owned.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_int32, _vp,
                                      ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _vp,
                                      ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.POINTER(ctypes.c_uint64)]


# ---- byte layout of the exchanges (pure Python, CPU-tested) --------------------------------------
def stream_layout(lens: list[list[int]]) -> tuple[list[list[int]], list[int]]:
    """lens[src][dst] = bytes src sends dst -> (base[src][dst] = offset of that stream in dst's
    receive buffer, recv[dst] = receive bytes): dst concatenates the streams in src order, which
    is the all-to-all output order and the reference's provenance order."""
    n = len(lens)
    base = [[0] * n for _ in range(n)]
    recv = [0] * n
    for dst in range(n):
        for src in range(n):
            base[src][dst] = recv[dst]
            recv[dst] += lens[src][dst]
    return base, recv


def virtual_shards(plans: list[tuple[list[list[int]], list[int]]], dst: int) -> list[int]:
    """plans[src] = (vs[dst][piece] offsets within src's stream to dst, len[dst]) -> the
    shard_offsets of dst's receive buffer (one virtual shard per (src, piece), then the end)."""
    lens = [p[1] for p in plans]
    base, recv = stream_layout(lens)
    offs = []
    for src, (vs, _) in enumerate(plans):
        offs.extend(base[src][dst] + v for v in vs[dst])
    offs.append(recv[dst])
    return offs


def slab_rows(n_batches: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [t0, t1) owned by `rank`: owner(t) = t * world // n_batches (route.cu tuple_owner)."""
    first = lambda r: min(n_batches, (r * n_batches + world - 1) // world)  # noqa: E731
    return first(rank), first(rank + 1)


def all_to_all_bytes(send: torch.Tensor, send_splits: list[int], recv_splits: list[int],
                     group=None) -> torch.Tensor:
    """uint8 all-to-all: NCCL on device tensors; gloo (tests: several ranks on one GPU) through
    host memory. Output is ordered by source rank."""
    dev = send.device
    on_cpu = dist.get_backend(group) == "gloo"
    s = send.cpu() if on_cpu else send
    recv = torch.empty(sum(recv_splits), dtype=torch.uint8, device="cpu" if on_cpu else dev)
    dist.all_to_all_single(recv, s, recv_splits, send_splits, group=group)
    return recv.to(dev) if on_cpu else recv


def all_gather_obj(obj, group=None) -> list:
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def agreed(fn, group=None):
    """Runs a rank-local step; every rank learns whether any rank failed and raises the same
    CvlError, so no rank is left waiting in the next collective."""
    err = None
    res = None
    try:
        res = fn()
    except _c.CvlError as e:
        err = (e.status, str(e))
    errs = [e for e in all_gather_obj(err, group) if e is not None]
    if errs:
        raise _c.CvlError(*errs[0])
    return res


# ---- the pipeline ---------------------------------------------------------------------------------
class FileShardedPipeline:
    """cvl::run_pipeline over the ranks of a process group (one GPU each)."""

    def __init__(self, paths, spec: _c.GridSpec | None = None, rules: _c.FilterRules | None = None,
                 ctx: _c.Context | None = None, threads: int = 0, group=None):
        self.paths = [str(p) for p in paths]
        self.spec = spec or _c.GridSpec()
        self.rules = rules or _c.FilterRules()
        self.ctx = ctx or _c.default_context()
        self.threads = threads
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local_bytes = 0    # bytes of this rank's range (route input)
        self.recv_bytes = 0     # bytes this rank received (its journeys' lines + headers)
        self.local_parsed = 0
        self.bad_headers = 0
        self._staged = False

    # step 1 (files -> this rank's range in HBM, counted per owner)
    def stage(self) -> None:
        arr = (ctypes.c_char_p * max(len(self.paths), 1))(*[p.encode() for p in self.paths])
        n_pieces = ctypes.c_uint64()
        bad = ctypes.c_uint64()
        _c._check(_lib.cvlg_route_stage(self.ctx.handle, arr, len(self.paths), self.world,
                                        self.rank, self.threads, ctypes.byref(n_pieces),
                                        ctypes.byref(bad)))
        self.n_pieces = n_pieces.value
        self.bad_headers = bad.value
        self._staged = True

    def _plan(self):
        vs, lens = [], []
        for o in range(self.world):
            offs = (ctypes.c_uint64 * max(self.n_pieces, 1))()
            ln = ctypes.c_uint64()
            _c._check(_lib.cvlg_route_plan(self.ctx.handle, o, offs, ctypes.byref(ln)))
            vs.append([int(offs[i]) for i in range(self.n_pieces)])
            lens.append(int(ln.value))
        return vs, lens

    def _run_staged(self, d_planes: torch.Tensor, d_raw: torch.Tensor | None) -> dict:
        dev = torch.device("cuda", torch.cuda.current_device())
        stream = torch.cuda.current_stream(dev).cuda_stream
        spec, world, g = self.spec, self.world, self.group
        T, D, R, C = spec.dims()
        # 2. route: send buffer partitioned by owner, all-to-all, virtual shards
        vs, lens = agreed(self._plan, g)
        plans = all_gather_obj((vs, lens), g)
        send_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        send = torch.empty(int(send_off[-1]) + 16, dtype=torch.uint8, device=dev)
        dst = (_vp * world)(*[send.data_ptr() + int(send_off[o]) for o in range(world)])
        torch.cuda.current_stream(dev).synchronize()
        _c._check(_lib.cvlg_route_scatter(self.ctx.handle, dst, None))
        recv_splits = [p[1][self.rank] for p in plans]
        recv = all_to_all_bytes(send[: int(send_off[-1])], lens, recv_splits, g)
        self.recv_bytes = recv.numel()
        self.local_bytes = recv.numel()  # what K1 decodes on this rank
        buf = torch.empty(recv.numel() + 16, dtype=torch.uint8, device=dev)
        buf[: recv.numel()].copy_(recv)
        del recv, send
        offs = virtual_shards(plans, self.rank)
        # 3. this rank's journeys up to the subtotals
        carr = (ctypes.c_uint64 * len(offs))(*offs)
        n_pairs = ctypes.c_uint64()
        st = _c._Stats()
        torch.cuda.current_stream(dev).synchronize()
        counts = (ctypes.c_uint64 * world)()
        n_t = ctypes.c_uint64()

        long_ids = ctypes.c_int32()

        def local():
            _c._check(_lib.cvlg_partial_device(self.ctx.handle, _vp(buf.data_ptr()), carr,
                                               len(offs) - 1, ctypes.byref(spec._c()),
                                               ctypes.byref(self.rules._c()), ctypes.byref(n_pairs),
                                               ctypes.byref(st), None))
            _c._check(_lib.cvlg_partial_info(self.ctx.handle, None, None, ctypes.byref(long_ids)))
        agreed(local, g)
        # 4. journey keys: exact inline ids, or global ranks when any rank has ids > 15 bytes
        grank = None
        if any(all_gather_obj(int(long_ids.value), g)):
            lists = all_gather_obj(self._journey_ids(), g)
            grank = self._merge(lists)[self.rank]
        agreed(lambda: _c._check(_lib.cvlg_tuples_export(
            self.ctx.handle, ctypes.byref(spec._c()), world,
            grank.ctypes.data_as(_vp) if grank is not None and grank.size else None,
            counts, ctypes.byref(n_t))), g)
        self.local_parsed = int(st.parsed)
        tcount = [int(counts[i]) for i in range(world)]
        toff = np.concatenate([[0], np.cumsum(tcount)]).astype(np.int64)
        tsend = torch.empty(int(toff[-1]) * TUPLE_BYTES + 64, dtype=torch.uint8, device=dev)
        tdst = (_vp * world)(*[tsend.data_ptr() + int(toff[s]) * TUPLE_BYTES for s in range(world)])
        _c._check(_lib.cvlg_tuples_scatter(self.ctx.handle, ctypes.byref(spec._c()), world, tdst,
                                           None))
        all_counts = all_gather_obj(tcount, g)
        trecv_splits = [c[self.rank] * TUPLE_BYTES for c in all_counts]
        trecv = all_to_all_bytes(tsend[: int(toff[-1]) * TUPLE_BYTES],
                                 [c * TUPLE_BYTES for c in tcount], trecv_splits, g)
        # 5. fold this rank's slab, all-gather the slabs
        n_in = trecv.numel() // TUPLE_BYTES
        rows = max(slab_rows(T, world, r)[1] - slab_rows(T, world, r)[0] for r in range(world))
        t0, t1 = slab_rows(T, world, self.rank)
        # this rank's slab rows, planes then raw counts per row (one buffer for the gather)
        mine = torch.zeros((max(rows, 1), 12, R, C), dtype=torch.int32, device=dev)
        slab_p = torch.empty((max(t1 - t0, 1), 8, R, C), dtype=torch.int32, device=dev)
        slab_r = torch.empty((max(t1 - t0, 1), 4, R, C), dtype=torch.int32, device=dev)
        _c._check(_lib.cvlg_finalize_tuples(self.ctx.handle, _vp(trecv.data_ptr()) if n_in else None,
                                            n_in, ctypes.byref(spec._c()), t0, t1,
                                            _vp(slab_p.data_ptr()), _vp(slab_r.data_ptr()),
                                            _vp(stream)))
        if t1 > t0:
            mine[: t1 - t0, :8].copy_(slab_p[: t1 - t0])
            mine[: t1 - t0, 8:].copy_(slab_r[: t1 - t0])
        gathered = self._all_gather(mine)
        for r in range(world):
            a, b = slab_rows(T, world, r)
            if b > a:
                d_planes[a:b].copy_(gathered[r][: b - a, :8])
                if d_raw is not None:
                    d_raw[a:b].copy_(gathered[r][: b - a, 8:])
        # stats: sum over ranks (+ BadHeader once)
        vals = [st.rows_read, st.parsed, st.duplicates_dropped, st.conflicting_duplicates,
                st.accepted, *st.rejected, *st.filtered]
        if self.rank == 0:
            vals[5 + 4] += self.bad_headers
        t = torch.tensor(vals, dtype=torch.int64)
        t = t.to(dev) if dist.get_backend(g) == "nccl" else t
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=g)
        v = [int(x) for x in t.cpu().tolist()]
        out = dict(zip(STAT_KEYS, v[:5]))
        out["rejected"] = {k: x for k, x in zip(_c.REJECT_NAMES, v[5:10]) if x}
        out["filtered"] = dict(zip(_c.FILTER_NAMES, v[10:13]))
        return out

    def _journey_ids(self) -> tuple[bytes, np.ndarray]:
        """This rank's journey ids in local rank order: (bytes, offsets[J + 1])."""
        nj, nb = ctypes.c_uint64(), ctypes.c_uint64()
        _c._check(_lib.cvlg_journey_ids(self.ctx.handle, None, 0, None, 0, ctypes.byref(nj),
                                        ctypes.byref(nb)))
        blob = np.empty(max(nb.value, 1), dtype=np.uint8)
        offs = np.empty(nj.value + 1, dtype=np.uint64)
        _c._check(_lib.cvlg_journey_ids(self.ctx.handle, blob.ctypes.data_as(_vp), blob.size,
                                        offs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                        offs.size, None, None))
        return blob[: nb.value].tobytes(), offs

    @staticmethod
    def _merge(lists) -> list[np.ndarray]:
        """Global lexicographic ranks of every rank's ids (cvlg_merge_id_ranks, host code)."""
        n = len(lists)
        blobs = [np.frombuffer(b or b"\0", dtype=np.uint8) for b, _ in lists]
        offs = [np.ascontiguousarray(o, dtype=np.uint64) for _, o in lists]
        ranks = [np.empty(max(len(o) - 1, 1), dtype=np.uint32) for o in offs]
        counts = (ctypes.c_uint64 * n)(*[len(o) - 1 for o in offs])
        _c._check(_lib.cvlg_merge_id_ranks(
            n, (_vp * n)(*[b.ctypes.data for b in blobs]), (_vp * n)(*[o.ctypes.data for o in offs]),
            counts, (_vp * n)(*[r.ctypes.data for r in ranks])))
        return [r[: len(o) - 1] for r, o in zip(ranks, offs)]

    def _all_gather(self, x: torch.Tensor) -> list[torch.Tensor]:
        g = self.group
        if dist.get_backend(g) == "gloo":
            parts = [torch.empty_like(x, device="cpu") for _ in range(self.world)]
            dist.all_gather(parts, x.cpu(), group=g)
            return [p.to(x.device) for p in parts]
        out = torch.empty((self.world, *x.shape), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x, group=g)
        return list(out)

    def run_files(self, out: tuple | None = None, stats: _c.PipelineStats | None = None):
        """End to end: shard files -> lattice in host memory on every rank."""
        agreed(self.stage, self.group)
        return self._finish(out, stats)

    def run_resident(self, d_planes: torch.Tensor, d_raw: torch.Tensor | None = None,
                     stats: _c.PipelineStats | None = None) -> None:
        """From this rank's range already in HBM (after run_files/stage): route ... combine."""
        if not self._staged:
            agreed(self.stage, self.group)
        else:
            agreed(lambda: _c._check(_lib.cvlg_route_count(self.ctx.handle)), self.group)
        st = self._run_staged(d_planes, d_raw)
        self._fill(stats, st)

    def _finish(self, out, stats):
        T, _, R, C = self.spec.dims()
        dev = torch.device("cuda", torch.cuda.current_device())
        d_planes = torch.empty((T, 8, R, C), dtype=torch.int32, device=dev)
        d_raw = torch.empty((T, 4, R, C), dtype=torch.int32, device=dev)
        st = self._run_staged(d_planes, d_raw)
        self._fill(stats, st)
        if out is None:
            planes = np.empty((T, 8, R, C), dtype=np.uint32)
            raw = np.empty((T, 4, R, C), dtype=np.uint32)
        else:
            planes, raw = out
        planes.view(np.int32)[...] = d_planes.cpu().numpy()
        if raw is not None:
            raw.view(np.int32)[...] = d_raw.cpu().numpy()
        return _c.Lattice(planes, raw)

    @staticmethod
    def _fill(stats, st: dict) -> None:
        if stats is None:
            return
        if isinstance(stats, dict):
            stats.clear()
            stats.update(st)
            return
        stats.rows_read = st["rows_read"]
        stats.parsed = st["parsed"]
        stats.duplicates_dropped = st["duplicates_dropped"]
        stats.conflicting_duplicates = st["conflicting_duplicates"]
        stats.accepted = st["accepted"]
        stats.rejected = dict(st["rejected"])
        stats.filtered = dict(st["filtered"])


def synth_day_owned(seed: int, journeys: int, shards: int, mean_duration: float, mod: int,
                    rem: int, sample_period: float = 1.0, day: str = "2021-05-09"):
    """The share of a `journeys`-journey synthetic day owned by rank `rem` of `mod` (generator
    side routing by the same FNV-1a; bench/test helper)."""
    import datetime
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

