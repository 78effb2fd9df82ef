#!/bin/bash
# one ncu --set full capture of decode_kernel on c2 (source-level counters)
TAG=${1:-prof}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -c 1 -o gpurun_out/$TAG python tools/profile_step.py --steps 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
