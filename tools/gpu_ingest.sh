#!/bin/bash
# Ingest probes: ring geometry sweep (page cache on /tmp) and zero-copy registration of tmpfs files.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out tools/_build
out=gpurun_out/ingest.log; : > $out
df -h /dev/shm /tmp >> $out 2>&1; mount | grep -E " /tmp | /dev/shm " >> $out
nvcc -O2 -o tools/_build/mmap_probe tools/mmap_probe.cu >> $out 2>&1
timeout 600 python tools/ring_sweep.py --reps 5 --grid "4:16,4:32,8:8,8:16,8:32,16:8,16:16,32:16" --threads 6,8,12 >> $out 2>&1
mkdir -p /dev/shm/probe && cp /tmp/cvlg_probe/j100000/shard_*.csv /dev/shm/probe/ && \
  timeout 300 tools/_build/mmap_probe /dev/shm/probe 16 >> $out 2>&1
timeout 300 tools/_build/mmap_probe /tmp/cvlg_probe/j100000 16 >> $out 2>&1
rm -rf /dev/shm/probe
cat $out
