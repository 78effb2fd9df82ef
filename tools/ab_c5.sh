#!/bin/bash
# A/B of library variants on c2 bench and c5-shape profile step
cd "$GRAFT_REPO_ROOT"
cp paper_2305_07454_b200/lib/libcvlg.so /tmp/libcvlg_base.so
for v in base "$@"; do
  if [ $v = base ]; then cp /tmp/libcvlg_base.so paper_2305_07454_b200/lib/libcvlg.so; else cp _var/libcvlg_$v.so paper_2305_07454_b200/lib/libcvlg.so; fi
  echo "$v c2 $(timeout 300 python bench.py --no-cpu --no-e2e --no-features --steps 20 | grep -o '"stage_ms": {[^}]*}')"
  echo "$v c5 $(timeout 300 python tools/profile_step.py --days 7 --fine --steps 3 2>&1 | tail -1)"
done
cp /tmp/libcvlg_base.so paper_2305_07454_b200/lib/libcvlg.so
