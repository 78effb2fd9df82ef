#!/bin/bash
# One GPU round-trip: parity tests, smoke, bench, ncu launch list (results under gpurun_out/).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench.log; tail -1 gpurun_out/bench_ref.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"decode_kernel|fold_lane" -c 2 -o gpurun_out/full python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
timeout 300 python tools/h2d_bw.py > gpurun_out/h2d.log 2>&1
