#!/usr/bin/env python
"""Benchmark of the sm_100a CV-ETL hot path (decode -> sort/dedup -> filter -> bin -> aggregate
-> finalize), BASELINE.json metric "CV records/sec end-to-end ETL ... vs CPU ref".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full pass of the pipeline over the configs[1] workload (c2: synthetic 50M-point
trace, 100k journeys, default GridSpec) — records are the CSV data rows.
  value : records/s, CSV already resident in HBM (device-resident API), CUDA events on the
          pipeline's stream, max over ranks.
  e2e   : records/s through the C ABI with HOST buffers (pinned), H2D of the CSV and D2H of the
          lattice inside every step.
Multi-GPU (torchrun): weak scaling, each rank owns the journeys whose FNV-1a id hash maps to it
(ingest.cpp:287-301) and processes its own 100k-journey share.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CV records/sec end-to-end ETL (1/2/4/8 B200) and % of HBM roofline vs CPU ref"
UNIT = "records/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--journeys", type=int, default=100_000, help="journeys per rank (c2)")
    ap.add_argument("--shards", type=int, default=16)
    ap.add_argument("--mean-duration", type=float, default=500.0)
    ap.add_argument("--cpu-journeys", type=int, default=10_000,
                    help="bounded CPU sample for cpu_baseline / --impl reference")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--days", type=int, default=1,
                    help="c5 shape: N consecutive days (seeds 1..N, same journey ids every day; the "
                         "time bin ignores the date, so days fold onto one time-of-day lattice)")
    ap.add_argument("--fine", action="store_true",
                    help="c5 grid: 0.01 degree cells and 1-minute bins (1.78 G cells, 14 GB lattice)")
    ap.add_argument("--shuffled", action="store_true",
                    help="adversarial variant (SURVEY §8d): rows shuffled across shards, so the "
                         "full (rank, ts) sort path runs")
    ap.add_argument("--no-features", action="store_true",
                    help="skip the per-journey feature-table timing (extra key, not the metric)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (in-process NVML: the
    nvidia-smi CLI polling every 100 ms was measured to stall CUDA API calls by 20-30 ms).
    One sample at entry, one at exit, and one every `interval` seconds in between."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index: int, interval: float = 0.25):
        self.disabled = os.environ.get("CVLG_NO_CLOCKS") == "1"  # diagnostics only
        self.gpu = gpu_index
        self.interval = interval
        self.samples: list[tuple[float, float, int]] = []
        self._stop = threading.Event()
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[gpu_index]) if vis else gpu_index
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(phys)
        except Exception:
            self.nvml = None

    def sample(self):
        if not self.nvml or self.disabled:
            return
        n = self.nvml
        try:
            sm = n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)
            mx = n.nvmlDeviceGetMaxClockInfo(self.handle, n.NVML_CLOCK_SM)
            rs = n.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
            self.samples.append((float(sm), float(mx), int(rs)))
        except Exception:
            pass

    def _run(self):
        while not self._stop.wait(self.interval):
            self.sample()

    def __enter__(self):
        self.sample()
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *a):
        self.sample()
        self._stop.set()
        self.thread.join(timeout=5)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [s[0] for s in self.samples]
        mx = max(s[1] for s in self.samples)
        reasons = sorted({k for _, _, r in self.samples for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(sm), "source": "NVML in-process"}


def measured_peak_hbm() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


def generate(journeys: int, shards: int, mean_duration: float, seed: int, mod: int = 1,
             rem: int = 0, days: int = 1):
    from paper_2305_07454_b200.cvlg import synth_day
    if days > 1:  # c5 shape: day k uses seed + k and date + k; its shards follow day k-1's
        import datetime
        import numpy as np
        if mod != 1:
            raise SystemExit("--days > 1 is single-GPU only in this bench")
        blobs, offs, rows = [], [0], 0
        for k in range(days):
            d = (datetime.date(2021, 5, 9) + datetime.timedelta(days=k)).isoformat()
            b, o, r = synth_day(seed=seed + k, journeys=journeys, shards=shards,
                                mean_duration=mean_duration, day=d)
            base = offs[-1]
            offs.extend(base + int(x) for x in o[1:])
            blobs.append(b)
            rows += r
        return np.concatenate(blobs), offs, rows
    if mod == 1:
        return synth_day(seed=seed, journeys=journeys, shards=shards, mean_duration=mean_duration)
    from paper_2305_07454_b200.distributed import synth_day_owned
    return synth_day_owned(seed=seed, journeys=journeys * mod, shards=shards,
                           mean_duration=mean_duration, mod=mod, rem=rem)


def cpu_reference_sample(args, tmpdir: Path):
    """Bounded sample of the same workload written as shard files for the reference."""
    from paper_2305_07454_b200.cvlg import synth_day
    threads = os.cpu_count() or 1
    shards = max(args.shards, threads)
    blob, offs, rows = synth_day(seed=1, journeys=args.cpu_journeys, shards=shards,
                                 mean_duration=args.mean_duration)
    paths = []
    for i in range(len(offs) - 1):
        p = tmpdir / f"shard_{i:04d}.csv"
        p.write_bytes(blob[offs[i]:offs[i + 1]].tobytes())
        paths.append(str(p))
    return paths, rows, threads


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Ref
    import paper_2305_07454_b200 as cvlg
    spec = cvlg.GridSpec()
    with tempfile.TemporaryDirectory() as d:
        paths, rows, threads = cpu_reference_sample(args, Path(d))
        ref = Ref()
        for _ in range(args.warmup):
            ref.run_pipeline(paths, spec, None, n_partitions=2 * threads, n_threads=threads,
                             raw=False)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            ref.run_pipeline(paths, spec, None, n_partitions=2 * threads, n_threads=threads,
                             raw=False)
            times.append(time.perf_counter() - t0)
    ms = 1000.0 * sum(times) / len(times)
    value = rows / (ms / 1000.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c2 (bounded CPU sample: %d journeys, %d rows per step)" % (
            args.cpu_journeys, rows), "grid": "default GridSpec 46x67x288x4"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{rows} rows ({args.cpu_journeys} journeys, seed 1) per step; "
                                   f"cvl::run_pipeline, {2 * threads} partitions"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    # CVLG_FORCE_DIST=1 exercises the multi-GPU combine path on a single GPU (tests)
    use_dist = world > 1 or os.environ.get("CVLG_FORCE_DIST") == "1"
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2305_07454_b200 as cvlg

    spec = (cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1) if args.fine
            else cvlg.GridSpec())
    t_gen = time.perf_counter()
    blob, offs, rows = generate(args.journeys, args.shards, args.mean_duration, seed=1,
                                mod=world, rem=rank, days=args.days)
    if args.shuffled:
        from paper_2305_07454_b200.cvlg import shuffle_rows
        blob, offs = shuffle_rows(blob, offs, args.shards, seed=7)
    t_gen = time.perf_counter() - t_gen
    csv_bytes = int(offs[-1])
    bufs = [blob[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
    T, _, R, C = spec.dims()
    ctx = cvlg.Context(local)

    # ---- device-resident value ------------------------------------------------------------------
    d_csv = torch.from_numpy(blob).to(f"cuda:{local}")
    d_planes = torch.empty((T, 8, R, C), dtype=torch.int32, device=f"cuda:{local}")
    d_raw = torch.empty((T, 4, R, C), dtype=torch.int32, device=f"cuda:{local}")
    stream = torch.cuda.current_stream()
    st = cvlg.PipelineStats()

    if use_dist:
        from paper_2305_07454_b200.distributed import run_pipeline_distributed
        dstats: dict = {}

    def step():
        if not use_dist:
            cvlg.run_pipeline_device(d_csv.data_ptr(), offs, d_planes.data_ptr(), d_raw.data_ptr(),
                                     spec, stats=st, ctx=ctx, stream=stream.cuda_stream)
        else:
            p, r = run_pipeline_distributed(d_csv, offs, spec, ctx=ctx, stats=dstats)
            d_planes.copy_(p)
            d_raw.copy_(r)
            st.rows_read = dstats["rows_read"]
            st.parsed = dstats["parsed"]

    for _ in range(max(args.warmup, 3)):
        step()
    assert st.rows_read == rows, (st.rows_read, rows)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = cvlg.launch_count()
    decode_ms = []
    stage = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            s = ctx.stage_ms()
            decode_ms.append(s[4])
            stage.append(s[:4])
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = cvlg.launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    rows_t = torch.tensor([int(rows)], dtype=torch.int64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(rows_t, op=dist.ReduceOp.SUM)
    ms_max = float(ms_t.item())
    total_rows = int(rows_t.item())
    value = total_rows / (ms_max / 1000.0)

    # ---- e2e through the host-buffer C ABI --------------------------------------------------------
    e2e = None
    if not args.no_e2e and use_dist:
        host = torch.from_numpy(blob).pin_memory()
        for _ in range(max(args.warmup, 3)):
            d_csv.copy_(host, non_blocking=True)
            p, _r = run_pipeline_distributed(d_csv, offs, spec, ctx=ctx)
            p.cpu()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            d_csv.copy_(host, non_blocking=True)
            p, r = run_pipeline_distributed(d_csv, offs, spec, ctx=ctx)
            p.cpu()
            r.cpu()
        torch.cuda.synchronize()
        e2e_ms = 1000.0 * (time.perf_counter() - t0) / args.steps
        e_t = torch.tensor([e2e_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
        e2e_ms = float(e_t.item())
        e2e = {"value": total_rows / (e2e_ms / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": csv_bytes, "d2h_bytes_per_step": int(p.numel() * 4 + r.numel() * 4),
               "ms_per_step": e2e_ms, "pinned_host": True, "note": "per-rank H2D + NCCL combine + D2H"}
    if not args.no_e2e and not use_dist:
        cvlg.pin_host(blob)
        planes = np.empty((T, 8, R, C), dtype=np.uint32)
        raw = np.empty((T, 4, R, C), dtype=np.uint32)
        cvlg.pin_host(planes)
        cvlg.pin_host(raw)
        for _ in range(max(args.warmup, 3)):
            cvlg.run_pipeline_host(bufs, spec, ctx=ctx, out=(planes, raw))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            cvlg.run_pipeline_host(bufs, spec, ctx=ctx, out=(planes, raw))
        e2e_ms = 1000.0 * (time.perf_counter() - t0) / args.steps
        e_t = torch.tensor([e2e_ms], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
        e2e_ms = float(e_t.item())
        # parity of the two entry points on this input
        dev_planes = d_planes.cpu().numpy().view(np.uint32)
        assert np.array_equal(dev_planes, planes), "host and device entry points disagree"
        e2e = {"value": total_rows / (e2e_ms / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": csv_bytes, "d2h_bytes_per_step": planes.nbytes + raw.nbytes,
               "ms_per_step": e2e_ms, "pinned_host": True}
        cvlg.unpin_host(planes)
        cvlg.unpin_host(raw)
        cvlg.unpin_host(blob)

    # ---- per-journey feature table (north_star extension; extra key, not the headline metric) ---
    features = None
    if not args.no_features and not use_dist and rank == 0:
        for _ in range(2):
            cvlg.journey_features_device(d_csv.data_ptr(), offs, d_planes.data_ptr(), d_raw.data_ptr(),
                                         spec, stop_speed=5.0, ctx=ctx, stream=stream.cuda_stream,
                                         fetch=False)
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        fsteps = max(3, min(args.steps, 10))
        f0.record(stream)
        for _ in range(fsteps):
            nj = cvlg.journey_features_device(d_csv.data_ptr(), offs, d_planes.data_ptr(),
                                              d_raw.data_ptr(), spec, stop_speed=5.0, ctx=ctx,
                                              stream=stream.cuda_stream, fetch=False)
        f1.record(stream)
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1) / fsteps
        features = {"ms_per_step": fms, "records_per_s": rows / (fms / 1000.0), "journeys": int(nj),
                    "note": "pipeline + per-journey feature table + per-cell speed min/max "
                            "(not in the reference: parity vs tests/features_oracle.py)"}

    # ---- roofline of the dominant kernel (K1 decode) ---------------------------------------------
    peak, peak_kind = measured_peak_hbm()
    dec_ms = sum(decode_ms) / len(decode_ms)
    n_heads_est = None
    dec_bytes = csv_bytes + st.parsed * 28  # CSV read + ts/speed/code/line-offset columns written
    achieved = dec_bytes / (dec_ms / 1000.0) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "decode_traffic.json"
    if tfile.exists():
        try:
            tj = json.loads(tfile.read_text())
            # the capture holds for the workload it was taken on only
            if tj.get("csv_bytes") == csv_bytes:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    stage_avg = [sum(s[i] for s in stage) / len(stage) for i in range(4)]

    # ---- CPU baseline (reference, rank 0, N = 1 only) ---------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle.oracle import Ref
            with tempfile.TemporaryDirectory() as d:
                paths, crow, threads = cpu_reference_sample(args, Path(d))
                ref = Ref()
                ref.run_pipeline(paths, spec, None, 2 * threads, threads, raw=False)
                ts = []
                for _ in range(2):
                    t0 = time.perf_counter()
                    ref.run_pipeline(paths, spec, None, 2 * threads, threads, raw=False)
                    ts.append(time.perf_counter() - t0)
            cpu = {"value": crow / (sum(ts) / len(ts)), "unit": UNIT, "cores": threads,
                   "kind": "reference",
                   "sample": f"{crow} rows ({args.cpu_journeys} journeys of the same generator, "
                             f"seed 1), cvl::run_pipeline with {threads} threads / "
                             f"{2 * threads} partitions, mean of 2 warm runs"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator algorithm, byte-identical; seed 1)",
            "config": {
                "workload": (f"c5 shape on 1 GPU: {args.days} consecutive days x {args.journeys} "
                             "journeys (same ids every day), device-resident"
                             if args.days > 1 else
                             "c2: synthetic 50M-point trace, 100k journeys per GPU, device-resident"
                             if args.journeys == 100_000 else
                             f"synthetic trace, {args.journeys} journeys per GPU "
                             f"(c3 = 1,000,000: full-day statewide shape), device-resident")
                            + (" | ADVERSARIAL: rows shuffled across shards (full-sort path)"
                               if args.shuffled else "")
                            + (" | fine 1-minute / 0.01 deg lattice" if args.fine else ""),
                "journeys_per_gpu": args.journeys, "rows_per_gpu": rows, "rows_total": total_rows,
                "csv_bytes_per_gpu": csv_bytes, "shards": args.shards,
                "grid": ("c5 fine grid: 0.01 deg cells, 1-minute bins (T=1440, 460x670: "
                         f"{1440 * 4 * 460 * 670:,} cells)" if args.fine
                         else "default GridSpec 46x67x288x4 (3,550,464 cells)"),
                "l2": "inputs (%.2f GB) larger than L2 (126 MB); no flush needed" % (csv_bytes / 1e9),
                "parallelism": f"dp{world} (journey-hash shards)",
                "input_generation_s": round(t_gen, 2),
            },
            "e2e": e2e,
            "roofline": {"bound": "hbm", "kernel": "decode_kernel (K1)", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": dec_bytes, "avg_launch_ms": dec_ms},
            "stage_ms": dict(zip(["decode", "dictionary+order", "fold", "finalize"], stage_avg)),
            "pipeline_hbm_frac": value * (csv_bytes / rows) / 1e9 / peak,
            "cpu_baseline": cpu,
            "features": features,
            "clocks": clocks.summary(),
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
