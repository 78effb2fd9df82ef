#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e --no-features --steps 20 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' | tr '\n' ' '; echo
timeout 300 python bench.py --shuffled --no-cpu --no-e2e --no-features --steps 5 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' | tr '\n' ' '; echo
timeout 300 python tools/profile_step.py --days 7 --fine --steps 2 2>&1 | tail -1
