#!/bin/bash
# ncu --set full of one big one-sweep radix pass (the shuffled c2 slot sort)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:radix_onesweep --launch-skip 16 -c 1 -o gpurun_out/sort_shuf python tools/profile_step.py --steps 1 --shuffle > gpurun_out/ncu_sort.log 2>&1
tail -n 2 gpurun_out/ncu_sort.log
