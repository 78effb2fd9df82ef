#!/bin/bash
# fold time-bin windows: new parity tests first, then c2/c5 stage times with windows on and off
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 200 python tools/profile_step.py --days 7 --fine --steps 2 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${1:-fine_grid or multi_day or c5_shape}" > gpurun_out/pytest_win.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_win.log
tail -5 gpurun_out/pytest_win.log
timeout 300 python bench.py --no-cpu --no-features --no-e2e --steps 10 | grep -o "\"ms_per_step\": [0-9.]*\|\"stage_ms\": {[^}]*}"
