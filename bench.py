#!/usr/bin/env python
"""Benchmark of the sm_100a CV-ETL hot path (decode -> sort/dedup -> filter -> bin -> aggregate
-> finalize), BASELINE.json metric "CV records/sec end-to-end ETL ... vs CPU ref".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3|c2]

Workload (default c3 = BASELINE.json configs[2], the largest single-GPU config): the reference
generator's full-day statewide-shaped trace, 1,000,000 journeys (~499M rows, ~33.8 GB of CSV),
seed 1, mean_duration 500 s, written as 128 shard files (the generator's own format and names,
synth.cpp:145-181). Records are the CSV data rows; one step = one full pass of the pipeline over
the whole trace.
  e2e   : records/s through the drop-in C ABI cvlg_run_pipeline(paths) (= cvl::run_pipeline,
          aggregate.hpp:125-127): shard files read from the file system (page cache) through the
          pinned ingest ring, H2D, decode ... finalize, and the D2H of the lattice, every step.
  value : records/s of the same pipeline on the same input already resident in HBM (the bytes
          the e2e run staged; cvlg_run_pipeline_device), CUDA events on the pipeline stream.
At N > 1 (c4: the same trace sharded by journey-id hash, strong scaling) every rank streams a
1/N byte range of the files and records are routed to their owner GPU (multi-GPU data plane).

Reference arm (--impl reference): the UNMODIFIED reference cvl::run_pipeline (oracle/_ref, built
from /root/reference/proj/src) on the SAME shard files, all host threads. It never imports this
package (its input is written by the reference's own generate_journey when absent). Each step
is a bounded sample: one eighth of the manifest (every 8th shard; journeys are dealt round-robin
to shards, synth.cpp:165, so each eighth is a uniform 1/8 of the journeys), cycling so that 8
steps cover the whole trace.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CV records/sec end-to-end ETL (1/2/4/8 B200) and % of HBM roofline vs CPU ref"
UNIT = "records/s"
GROUPS = 8  # the reference arm's bounded sample: one eighth of the manifest per step

WORKLOADS = {
    "c3": dict(journeys=1_000_000, shards=128, seed=1, mean_duration=500.0,
               desc="c3: full-day statewide-shaped synthetic trace (1,000,000 journeys), "
                    "end-to-end from shard files incl. disk->pinned->H2D"),
    "c2": dict(journeys=100_000, shards=128, seed=1, mean_duration=500.0,
               desc="c2: synthetic 50M-point trace, 100k journeys"),
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--data-dir", default=os.environ.get("CVLG_BENCH_DATA", "/tmp/cvlg_bench"))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the sampled parity check")
    ap.add_argument("--threads", type=int, default=0, help="host threads (0 = all)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def maybe_relaunch(args):
    """--gpus N outside torchrun: re-exec under torch.distributed.run with N ranks."""
    world = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if args.gpus > 1 and world == 0:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={29500 + os.getpid() % 1000}", str(Path(__file__).resolve())]
        cmd += sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if world and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")


# ---- shared input: shard files on the file system ---------------------------------------------
def dataset_dir(args) -> Path:
    w = WORKLOADS[args.workload]
    return Path(args.data_dir) / f"{args.workload}_s{w['seed']}_j{w['journeys']}_n{w['shards']}"


def _digest(files: list[Path]) -> str:
    h = hashlib.sha256()
    for f in files:
        sz = f.stat().st_size
        h.update(f.name.encode() + sz.to_bytes(8, "little"))
        with open(f, "rb") as fh:
            h.update(fh.read(4096))
            if sz > 4096:
                fh.seek(max(4096, sz - 4096))
                h.update(fh.read(4096))
    return h.hexdigest()


def load_manifest(d: Path):
    m = d / "MANIFEST.json"
    if not m.exists():
        return None
    try:
        j = json.loads(m.read_text())
        files = [d / n for n, _ in j["files"]]
        if any(not f.exists() or f.stat().st_size != s for f, (_, s) in zip(files, j["files"])):
            return None
        if _digest(files) != j["digest"]:
            return None
        return j
    except Exception:
        return None


def ensure_dataset(args, generator) -> tuple[list[str], dict, float]:
    """Shard files of the workload (generated once per box, reused by both arms). `generator`
    (out_dir, seed, journeys, shards, mean_duration) -> rows writes generate_day's files."""
    w = WORKLOADS[args.workload]
    d = dataset_dir(args)
    man = load_manifest(d)
    t_gen = 0.0
    if man is None:
        root = Path(args.data_dir)
        root.mkdir(parents=True, exist_ok=True)
        for other in root.iterdir():  # one dataset at a time (disk space)
            if other.is_dir():
                shutil.rmtree(other, ignore_errors=True)
        tmp = root / (d.name + ".tmp")
        shutil.rmtree(tmp, ignore_errors=True)
        tmp.mkdir(parents=True)
        t0 = time.perf_counter()
        rows = generator(tmp, w["seed"], w["journeys"], w["shards"], w["mean_duration"])
        t_gen = time.perf_counter() - t0
        files = sorted(tmp.glob("shard_*.csv"))
        man = {"files": [[f.name, f.stat().st_size] for f in files], "rows": int(rows),
               "digest": _digest(files), "workload": args.workload, **{k: w[k] for k in
               ("journeys", "shards", "seed", "mean_duration")}}
        (tmp / "MANIFEST.json").write_text(json.dumps(man))
        os.replace(tmp, d)
    paths = [str(d / n) for n, _ in man["files"]]
    return paths, man, t_gen


def groups_of(paths: list[str]) -> list[list[str]]:
    return [[p for i, p in enumerate(paths) if i % GROUPS == g] for g in range(GROUPS)]


def config_of(args, man, world) -> dict:
    """Identical in both arms (the driver compares them)."""
    w = WORKLOADS[args.workload]
    wl = w["desc"] if world == 1 else (
        f"c4: the {args.workload} trace sharded by journey-id hash (FNV-1a % N) at {world} B200, "
        "end-to-end from shard files")
    return {
        "workload": wl, "journeys": w["journeys"], "rows": man["rows"],
        "csv_bytes": sum(s for _, s in man["files"]), "shards": w["shards"], "seed": w["seed"],
        "mean_duration_s": w["mean_duration"],
        "grid": "default GridSpec 46x67x288x4 (3,550,464 cells)",
        "l2": "inputs (%.1f GB) larger than L2 (126 MB); no flush needed"
              % (sum(s for _, s in man["files"]) / 1e9),
        "parallelism": f"dp{world} (journey-hash shards)",
    }


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (in-process NVML)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index: int, interval: float = 0.25):
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
        if not self.nvml:
            return
        n = self.nvml
        try:
            self.samples.append((float(n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)),
                                 float(n.nvmlDeviceGetMaxClockInfo(self.handle, n.NVML_CLOCK_SM)),
                                 int(n.nvmlDeviceGetCurrentClocksEventReasons(self.handle))))
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
        reasons = sorted({k for _, _, r in self.samples for k, b in self.REASONS.items() if r & b})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "NVML in-process"}


def measured_peak_hbm() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def lattice_sha(planes, raw) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(planes).view(np.uint8))
    if raw is not None:
        h.update(np.ascontiguousarray(raw).view(np.uint8))
    return h.hexdigest()


# ---- reference arm -----------------------------------------------------------------------------
def ref_generator(threads):
    from oracle.oracle import Ref

    def gen(out, seed, journeys, shards, mean_duration):
        return Ref().generate_day_mt(out, seed=seed, journeys=journeys, shards=shards,
                                     mean_duration=mean_duration, threads=threads)
    return gen


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    assert "paper_2305_07454_b200" not in sys.modules
    from oracle.oracle import Ref, CGrid  # noqa: F401  (the compiled, unmodified reference)

    class Spec:  # the default GridSpec (grid.hpp:21-41)
        lat_min, lat_max, lon_min, lon_max = 36.0, 40.6, -95.8, -89.1
        lat_step = lon_step = 0.1
        min_step, dxn_step, dxn_offset = 5, 90, 0.0

    threads = args.threads or os.cpu_count() or 1
    paths, man, t_gen = ensure_dataset(args, ref_generator(threads))
    groups = groups_of(paths)
    ref = Ref()
    rows_of = {}

    def step(i):
        g = groups[i % GROUPS]
        _, _, st, _ = ref.run_pipeline(g, Spec, None, n_partitions=2 * threads,
                                       n_threads=threads, raw=False)
        rows_of[i % GROUPS] = st["rows_read"]
        return st["rows_read"]

    for i in range(args.warmup):
        step(i)
    rows = 0
    t0 = time.perf_counter()
    for i in range(args.steps):
        rows += step(args.warmup + i)
    dt = time.perf_counter() - t0
    value = rows / dt
    sample = (f"cvl::run_pipeline (unmodified, oracle/_ref) with {threads} threads / "
              f"{2 * threads} partitions; each step = 1/{GROUPS} of the same {len(paths)}-shard "
              f"manifest (every {GROUPS}th shard, ~{rows / max(args.steps, 1) / 1e6:.1f}M rows), "
              f"cycling over the {GROUPS} eighths; {rows} rows in {args.steps} timed steps")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, seed 1), shard files on the local file system",
        "config": config_of(args, man, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "input_generation_s": round(t_gen, 1),
    }
    print(json.dumps(line), flush=True)


# ---- our arm -----------------------------------------------------------------------------------
def our_generator(threads):
    from paper_2305_07454_b200.cvlg import synth_write_day

    def gen(out, seed, journeys, shards, mean_duration):
        return synth_write_day(out, seed=seed, journeys=journeys, shards=shards,
                               mean_duration=mean_duration, threads=threads)[1]
    return gen


def cpu_baseline_leg(args, paths, spec_ref):
    """The reference on one eighth of the same files (rank 0, N = 1): ~10-30 s of CPU work."""
    from oracle.oracle import Ref
    threads = args.threads or os.cpu_count() or 1
    g = groups_of(paths)[0]
    ref = Ref()
    ref.run_pipeline(g, spec_ref, None, 2 * threads, threads, raw=False)
    ts, out = [], None
    for _ in range(2):
        t0 = time.perf_counter()
        out = ref.run_pipeline(g, spec_ref, None, 2 * threads, threads, raw=True)
        ts.append(time.perf_counter() - t0)
    planes, raw, st, _ = out
    cpu = {"value": st["rows_read"] / (sum(ts) / len(ts)), "unit": UNIT, "cores": threads,
           "kind": "reference",
           "sample": f"{st['rows_read']} rows = shards 0,8,16,... (1/{GROUPS}) of the same "
                     f"manifest; cvl::run_pipeline (unmodified) with {threads} threads / "
                     f"{2 * threads} partitions, mean of 2 warm runs"}
    return cpu, g, planes, raw, st


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # (CVLG_BENCH_DEVICE / CVLG_BENCH_BACKEND: exercise the N-rank path on fewer GPUs, e.g. two
    # ranks sharing cuda:0 over gloo; never used for a reported number)
    if os.environ.get("CVLG_BENCH_DEVICE"):
        local = int(os.environ["CVLG_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("CVLG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2305_07454_b200 as cvlg

    threads = args.threads or os.cpu_count() or 1
    if world > 1:
        threads = max(1, threads // world)
    if rank == 0:
        paths, man, t_gen = ensure_dataset(args, our_generator(threads))
    if world > 1:
        dist.barrier()
        if rank != 0:
            paths, man, t_gen = ensure_dataset(args, our_generator(threads))
    rows = man["rows"]
    csv_bytes = sum(s for _, s in man["files"])
    spec = cvlg.GridSpec()
    T, _, R, C = spec.dims()
    ctx = cvlg.Context(local)
    planes = np.empty((T, 8, R, C), dtype=np.uint32)
    raw = np.empty((T, 4, R, C), dtype=np.uint32)
    cvlg.pin_host(planes)
    cvlg.pin_host(raw)
    st = cvlg.PipelineStats()

    if world > 1:
        from paper_2305_07454_b200.distributed import FileShardedPipeline
        runner = FileShardedPipeline(paths, spec, ctx=ctx, threads=threads)
        e2e_step = lambda: runner.run_files(out=(planes, raw), stats=st)  # noqa: E731
    else:
        e2e_step = lambda: cvlg.run_pipeline(paths, spec, n_partitions=2 * threads,  # noqa: E731
                                             n_threads=threads, stats=st, ctx=ctx,
                                             out=(planes, raw))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        on_dev = dist.get_backend() == "nccl"
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}" if on_dev else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- e2e through the drop-in C ABI (files -> lattice in host memory) ---------------------
    for _ in range(max(args.warmup, 3)):
        e2e_step()
    assert st.rows_read == rows, (st.rows_read, rows)
    e2e_sha = lattice_sha(planes, raw)
    barrier()
    torch.cuda.synchronize()
    e2e = None
    e2e_clocks = None
    if not args.no_e2e:
        with ClockSampler(local) as ck:
            t0 = time.perf_counter()
            for _ in range(args.steps):
                e2e_step()
            torch.cuda.synchronize()
            e2e_s = time.perf_counter() - t0
        e2e_clocks = ck.summary()
        barrier()
        e2e_ms = max_over_ranks(1000.0 * e2e_s / args.steps)
        e2e = {"value": rows / (e2e_ms / 1000.0), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": csv_bytes,
               "d2h_bytes_per_step": int(planes.nbytes + raw.nbytes),
               "path": "cvlg_run_pipeline(shard paths): pread (page cache) -> pinned ring -> H2D "
                       "-> pipeline -> D2H of the lattice, every step"}

    # ---- device-resident value: the same bytes, already in HBM --------------------------------
    stream = torch.cuda.current_stream()
    d_planes = torch.empty((T, 8, R, C), dtype=torch.int32, device=f"cuda:{local}")
    d_raw = torch.empty((T, 4, R, C), dtype=torch.int32, device=f"cuda:{local}")
    if world > 1:
        dev_step = lambda: runner.run_resident(d_planes, d_raw, stats=st)  # noqa: E731
    else:
        d_csv, n_in = ctx.input()
        assert n_in == csv_bytes
        offs = [0]
        for _, s in man["files"]:
            offs.append(offs[-1] + s)
        dev_step = lambda: cvlg.run_pipeline_device(d_csv, offs, d_planes.data_ptr(),  # noqa: E731
                                                    d_raw.data_ptr(), spec, stats=st, ctx=ctx,
                                                    stream=stream.cuda_stream)
    for _ in range(max(args.warmup, 3)):
        dev_step()
    dev_sha = lattice_sha(d_planes.cpu().numpy().view(np.uint32), d_raw.cpu().numpy().view(np.uint32))
    assert dev_sha == e2e_sha, "file and device-resident entry points disagree"
    barrier()
    torch.cuda.synchronize()
    launches0 = cvlg.launch_count()
    stage, decode_ms = [], []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            dev_step()
            s = ctx.stage_ms()
            stage.append(s[:4])
            decode_ms.append(s[4])
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = cvlg.launch_count() - launches0
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    value = rows / (ms / 1000.0)

    # ---- roofline of the dominant kernel (K1 decode) ------------------------------------------
    peak, peak_kind = measured_peak_hbm()
    dec_ms = sum(decode_ms) / len(decode_ms)
    local_bytes = csv_bytes if world == 1 else runner.local_bytes
    local_parsed = st.parsed if world == 1 else runner.local_parsed
    dec_bytes = local_bytes + local_parsed * 28  # CSV read + 28 B/slot of columns written
    achieved = dec_bytes / (dec_ms / 1000.0) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "decode_traffic.json"
    if tfile.exists() and world == 1:  # (the device-resident run is one K1 launch over the input)
        try:
            tj = json.loads(tfile.read_text())
            for e in (tj if isinstance(tj, list) else [tj]):
                if e.get("csv_bytes") == local_bytes:
                    traffic = e.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    stage_avg = [sum(s[i] for s in stage) / len(stage) for i in range(4)]

    # ---- CPU baseline + sampled parity (reference, rank 0, N = 1 only) ------------------------
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        class SpecRef:
            lat_min, lat_max, lon_min, lon_max = 36.0, 40.6, -95.8, -89.1
            lat_step = lon_step = 0.1
            min_step, dxn_step, dxn_offset = 5, 90, 0.0
        try:
            cpu, g, rp, rr, rst = cpu_baseline_leg(args, paths, SpecRef)
            if not args.no_parity:
                gst = cvlg.PipelineStats()
                lat = cvlg.run_pipeline(g, spec, n_partitions=1, n_threads=threads, stats=gst,
                                        ctx=ctx)
                same = (np.array_equal(lat.planes, rp) and np.array_equal(lat.raw, rr)
                        and gst.rows_read == rst["rows_read"] and gst.parsed == rst["parsed"]
                        and gst.accepted == rst["accepted"])
                parity = {"sample": f"1/{GROUPS} of the manifest ({rst['rows_read']} rows)",
                          "vs": "cvl::run_pipeline (unmodified)",
                          "lattice_and_stats_bit_identical": bool(same),
                          "lattice_sha256": lattice_sha(lat.planes, lat.raw)}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, seed 1), shard files on the local file system",
            "config": config_of(args, man, world),
            "e2e": e2e,
            "roofline": {"bound": "hbm", "kernel": "decode_kernel (K1)", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch_sum": dec_bytes, "avg_decode_ms": dec_ms},
            "stage_ms": dict(zip(["parse", "dedup+filter+accumulate", "merge", "finalize"],
                                 stage_avg)),
            "pipeline_hbm_frac": value * (csv_bytes / rows) / 1e9 / peak,
            "cpu_baseline": cpu,
            "parity_sample": parity,
            "lattice_sha256": e2e_sha,
            "clocks": clocks.summary(),
            "e2e_clocks": e2e_clocks,
            "gpu_launches": launches,
            "input_generation_s": round(t_gen, 1),
        }
        print(json.dumps(line), flush=True)
    cvlg.unpin_host(planes)
    cvlg.unpin_host(raw)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    maybe_relaunch(args)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
