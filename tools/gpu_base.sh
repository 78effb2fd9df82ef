#!/bin/bash
# Round-2 baseline: parity tests, ncu --set full of K1 (c2), launch list (c2), bench c3 + c2.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${1:-decode_kernel}" -c 1 -o gpurun_out/prof python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 900 python bench.py --workload c2 --steps 10 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c2.log
timeout 1200 python bench.py --steps 10 > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3.log
tail -4 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/ncu_full.log; tail -2 gpurun_out/bench_c2.log | cut -c1-400; tail -2 gpurun_out/bench_c3.log | cut -c1-400
