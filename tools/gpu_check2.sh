#!/bin/bash
# full GPU parity suite + secondary-path timings
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
tail -3 gpurun_out/pytest_full.log
bash tools/gpu_paths.sh
