#!/bin/bash
# parity tests, then one ncu --set full capture of the decode kernel (c2 workload)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${1:-decode_kernel}" -c 1 -o gpurun_out/prof python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -4 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/ncu_full.log; tail -2 gpurun_out/bench.log | cut -c1-600
