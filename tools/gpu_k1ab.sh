#!/bin/bash
# K1 A/B on one box: ncu counters of decode_kernel for each lib/libcvlg.<variant>.so and the
# current build, then the decode parity tests and a c2 bench.  usage: tools/gpu_k1ab.sh TAG [full]
TAG=${1:-ab}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_shared_mem
out=gpurun_out/ab_$TAG.txt; : > $out
for f in paper_2305_07454_b200/lib/libcvlg.*.so; do
  v=$(basename $f .so); v=${v#libcvlg.}
  CVLG_LIB_VARIANT=$v timeout 300 ncu --metrics $M --clock-control none -k regex:decode_kernel -c 2 python tools/profile_step.py --steps 2 > /tmp/ncu_$v.txt 2>&1
  echo "== $v" >> $out; grep -E "gpu__time|inst_executed|issue_active|warps_active|registers|occupancy" /tmp/ncu_$v.txt | tail -6 >> $out
done
timeout 300 ncu --metrics $M --clock-control none -k regex:decode_kernel -c 2 python tools/profile_step.py --steps 2 > /tmp/ncu_main.txt 2>&1
echo "== main" >> $out; grep -E "gpu__time|inst_executed|issue_active|warps_active|registers|occupancy" /tmp/ncu_main.txt | tail -6 >> $out
cat $out
if [ "$2" == "none" ]; then echo "tests skipped";
elif [ "$2" == "full" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
else
  timeout 900 python -m pytest tests/test_decode_slots.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
fi
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$TAG.log 2>&1
python - <<PY
import json
l=[x for x in open("gpurun_out/bench_$TAG.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("value", d["value"]/1e9, "G rec/s ms", d["ms_per_step"], "decode ms", d["roofline"]["avg_decode_ms"], "frac", d["roofline"]["frac"], d["stage_ms"])
else: print(open("gpurun_out/bench_$TAG.log").read()[-2000:])
PY
