#!/bin/bash
# A/B of library variants: _var/libcvlg_<name>.so against the in-tree build (c2 stage times)
cd "$GRAFT_REPO_ROOT"
cp paper_2305_07454_b200/lib/libcvlg.so /tmp/libcvlg_base.so
for v in base "$@"; do
  if [ $v = base ]; then cp /tmp/libcvlg_base.so paper_2305_07454_b200/lib/libcvlg.so; else cp _var/libcvlg_$v.so paper_2305_07454_b200/lib/libcvlg.so; fi
  for r in 1 2; do
    echo "$v $(timeout 300 python bench.py --no-cpu --no-e2e --no-features --steps 20 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' | tr '\n' ' ')"
  done
done
cp /tmp/libcvlg_base.so paper_2305_07454_b200/lib/libcvlg.so
