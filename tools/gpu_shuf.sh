#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-x}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
tail -2 gpurun_out/pytest_$TAG.log
bash tools/gpu_launches.sh $TAG > gpurun_out/launches_$TAG.txt 2>&1; head -16 gpurun_out/launches_$TAG.txt
