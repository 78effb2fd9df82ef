#!/bin/bash
# round 2: multi-GPU data plane tests + smoke
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_distributed.py tests/test_multi.py -m gpu -x -q > gpurun_out/pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multi.log
tail -3 gpurun_out/smoke.log; tail -30 gpurun_out/pytest_multi.log
