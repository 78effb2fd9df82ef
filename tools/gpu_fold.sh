#!/bin/bash
# fold iteration: GPU tests, ncu of the fold kernel at c2 and the fine multi-day shape, c2 bench
TAG=${1:-fold}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:fold_lane -c 2 python tools/profile_step.py --steps 2 > gpurun_out/ncu_${TAG}_c2.txt 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:fold_lane -c 2 python tools/profile_step.py --steps 2 --journeys 100000 --days 3 --fine > gpurun_out/ncu_${TAG}_fine.txt 2>&1
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$TAG.log 2>&1
tail -2 gpurun_out/pytest_$TAG.log
for f in c2 fine; do echo "== $f"; grep -E "gpu__time|inst_executed|issue_active|warps_active|dram__bytes" gpurun_out/ncu_${TAG}_$f.txt | tail -6; done
python - <<PY
import json
l=[x for x in open("gpurun_out/bench_$TAG.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("value", d["value"]/1e9, "G rec/s ms", d["ms_per_step"], d["stage_ms"])
else: print(open("gpurun_out/bench_$TAG.log").read()[-2000:])
PY
