#!/bin/bash
# A/B of an environment switch: c2 bench and c5-shape step with VAR=0 / VAR=1
cd "$GRAFT_REPO_ROOT"
var=$1
for v in 0 1; do
  echo "$var=$v c2 $(env $var=$v timeout 300 python bench.py --no-cpu --no-e2e --no-features --steps 20 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' | tr '\n' ' ')"
  echo "$var=$v c5 $(env $var=$v timeout 300 python bench.py --days 7 --fine --no-cpu --no-e2e --no-features --steps 3 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' | tr '\n' ' ')"
done
