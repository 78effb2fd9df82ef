#!/bin/bash
# ncu --set full of the fold on c2 and on few long journeys
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fold_lane -c 1 -o gpurun_out/fold_c2 python tools/profile_step.py --steps 1 > gpurun_out/ncu_fold_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fold_lane -c 1 -o gpurun_out/fold_long python tools/profile_step.py --steps 1 --journeys 1000 --mean-duration 36000 > gpurun_out/ncu_fold_long.log 2>&1
tail -1 gpurun_out/ncu_fold_c2.log gpurun_out/ncu_fold_long.log
