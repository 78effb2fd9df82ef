#!/bin/bash
# Round evidence: parity tests, smoke, bench (+ CPU baseline, reference arm, adversarial variant),
# launch list, one ncu --set full of decode and fold. Everything lands in gpurun_out/.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --shuffled --no-cpu --no-features --steps 10 > gpurun_out/bench_shuf.log 2>&1
timeout 900 python bench.py --days 7 --fine --no-cpu --no-features --steps 5 > gpurun_out/bench_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/profile_step.py --days 7 --fine --steps 1 > gpurun_out/c5_prof.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"decode_kernel|fold_lane" -c 2 -o gpurun_out/full python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench.log
