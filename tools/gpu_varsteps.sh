#!/bin/bash
# A/B of whole-step times: tools/profile_step.py ARGS for every lib/libcvlg.<variant>.so and main
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
out=gpurun_out/varsteps.log; : > $out
for a in "$@"; do
  for f in $(ls paper_2305_07454_b200/lib/libcvlg.*.so 2>/dev/null); do
    v=$(basename $f .so); v=${v#libcvlg.}
    echo "== $v [$a]: $(CVLG_LIB_VARIANT=$v timeout 600 python tools/profile_step.py $a 2>&1 | tail -1)" >> $out
  done
  echo "== main [$a]: $(timeout 600 python tools/profile_step.py $a 2>&1 | tail -1)" >> $out
done
cat $out
