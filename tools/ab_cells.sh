#!/bin/bash
# A/B of the fold's per-lane cell-table size (gpurun_out/var/libcvlg_<n>.so builds)
cd "$GRAFT_REPO_ROOT"
cp paper_2305_07454_b200/lib/libcvlg.so /tmp/libcvlg_16.so
for c in 16 12 8; do
  if [ $c = 16 ]; then cp /tmp/libcvlg_16.so paper_2305_07454_b200/lib/libcvlg.so; else cp gpurun_out/var/libcvlg_$c.so paper_2305_07454_b200/lib/libcvlg.so; fi
  echo "cells=$c $(python bench.py --no-cpu --no-e2e --steps 10 | grep -o '"stage_ms": {[^}]*}')"
done
cp /tmp/libcvlg_16.so paper_2305_07454_b200/lib/libcvlg.so
