#!/bin/bash
# K1 iteration: parity (decode-heavy tests), ncu counters of the decode kernel, c2 bench
# usage: bash tools/gpu_k1.sh TAG [full]
TAG=${1:-k1}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
if [ "$2" == "full" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
else
  timeout 900 python -m pytest tests/test_decode_slots.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
fi
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__occupancy_limit_shared_mem --clock-control none -k regex:decode_kernel -c 2 python tools/profile_step.py --steps 2 > gpurun_out/ncu_$TAG.txt 2>&1
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$TAG.log 2>&1
tail -2 gpurun_out/pytest_$TAG.log; grep -E "gpu__time|inst_executed|issue_active|warps_active|dram__bytes|registers|occupancy" gpurun_out/ncu_$TAG.txt | tail -9
python - <<PY
import json
l=[x for x in open("gpurun_out/bench_$TAG.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("value", d["value"]/1e9, "G rec/s ms", d["ms_per_step"], "decode ms", d["roofline"]["avg_decode_ms"], "frac", d["roofline"]["frac"], d["stage_ms"])
else: print(open("gpurun_out/bench_$TAG.log").read()[-2000:])
PY
