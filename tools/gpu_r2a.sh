#!/bin/bash
# round-2 first measurement: parity tests, c2 + c3 bench (files), reference arm, decode ncu
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; df -h /tmp /root) > gpurun_out/r2a_mem.txt
timeout 1200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -c 1 -o gpurun_out/r2a_decode python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 python bench.py --workload c2 --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
free -g >> gpurun_out/r2a_mem.txt
timeout 900 python bench.py --impl reference --steps 8 --warmup 1 > gpurun_out/bench_c3_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3_ref.log
tail -4 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/ncu_full.log; for f in bench_c2 bench_c3 bench_c3_ref; do tail -3 gpurun_out/$f.log | cut -c1-1500; done
