#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -4 gpurun_out/sanitize_$tool.log
done
