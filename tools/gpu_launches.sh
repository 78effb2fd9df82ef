#!/bin/bash
# per-kernel launch lists (ncu gpu__time_duration, serialized) for the c2 shuffled path and c2
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shuf_$TAG.csv python tools/profile_step.py --steps 1 --shuffle > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$TAG.csv python tools/profile_step.py --steps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_shuf_$TAG.csv | head -30
python tools/launch_summary.py gpurun_out/launches_c2_$TAG.csv | head -30
