#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nproc > gpurun_out/ring_sweep.log; lscpu | grep -E "Model name|NUMA|Socket|Thread|Core" >> gpurun_out/ring_sweep.log; free -g >> gpurun_out/ring_sweep.log; df -h /tmp >> gpurun_out/ring_sweep.log
timeout 900 python tools/ring_sweep.py --threads 8,16 >> gpurun_out/ring_sweep.log 2>&1
cat gpurun_out/ring_sweep.log
