#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in ""; do
  echo "== variant '$v'"
  CVLG_LIB_VARIANT=$v timeout 600 python tools/profile_step.py --steps 2 --journeys 100000 --days 3 --fine 2>&1 | tail -2
done

M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:fold_lane -c 2 python tools/profile_step.py --steps 2 --journeys 100000 --days 3 --fine 2>&1 | grep -E "gpu__time|inst_exec|issue_active|warps_active|dram__bytes" | tail -6
