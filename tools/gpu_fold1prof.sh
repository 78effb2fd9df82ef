#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fold_lane -c 1 -o gpurun_out/fold_shuf python tools/profile_step.py --steps 1 --shuffle > gpurun_out/ncu_fold_shuf.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_shuf.csv python tools/profile_step.py --steps 1 --shuffle > /dev/null 2>&1
tail -n 1 gpurun_out/ncu_fold_shuf.log
