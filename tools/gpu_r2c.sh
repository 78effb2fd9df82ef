#!/bin/bash
# round 2: per-slot decode parity, compute-sanitizer, ingest probe
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decode_slots.py -x -q > gpurun_out/pytest_slots.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slots.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
timeout 900 python tools/ingest_probe.py > gpurun_out/ingest_probe.log 2>&1; echo "rc=$?" >> gpurun_out/ingest_probe.log
tail -3 gpurun_out/pytest_slots.log; for t in memcheck racecheck synccheck; do tail -4 gpurun_out/sanitize_$t.log; done; cat gpurun_out/ingest_probe.log | tail -40
