#!/bin/bash
# full GPU parity suite + step timings (c2, shuffled c2, long journeys)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
tail -3 gpurun_out/pytest_full.log
bash tools/gpu_varsteps.sh "--steps 5" "--steps 5 --shuffle" "--steps 4 --journeys 1000 --mean-duration 36000"
