#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_records.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_records.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_records.log
tail -30 gpurun_out/pytest_records.log
