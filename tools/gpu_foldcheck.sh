#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -x -q -k "fine_grid or multi_day or c5_shape or partial_export or synth_day or golden" > gpurun_out/pytest_fold.log 2>&1; tail -1 gpurun_out/pytest_fold.log
echo "c2 $(timeout 300 python bench.py --no-cpu --no-e2e --no-features --steps 20 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' | tr '\n' ' ')"
echo "c5 $(timeout 300 python bench.py --days 7 --fine --no-cpu --no-e2e --no-features --steps 3 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' | tr '\n' ' ')"
