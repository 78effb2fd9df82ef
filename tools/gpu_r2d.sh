#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "
import sys; sys.path.insert(0,'.')
import paper_2305_07454_b200 as c
c.cvlg.synth_write_day('/tmp/probe_c2', seed=1, journeys=100000, shards=128, mean_duration=500.0)
" > gpurun_out/mmap_probe.log 2>&1
cat /tmp/probe_c2/*.csv > /dev/null
for t in 8 12 16; do timeout 600 tools/_build/mmap_probe /tmp/probe_c2 $t d >> gpurun_out/mmap_probe.log 2>&1; done; true >> gpurun_out/mmap_probe.log 2>&1

cat gpurun_out/mmap_probe.log
