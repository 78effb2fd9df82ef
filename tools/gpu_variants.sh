#!/bin/bash
# K1 A/B: ncu time + instructions of the decode kernel for each lib/libcvlg.<variant>.so
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
out=gpurun_out/variants_${1:-x}.txt; : > $out
for f in paper_2305_07454_b200/lib/libcvlg.*.so; do
  v=$(basename $f .so); v=${v#libcvlg.}
  CVLG_LIB_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:decode_kernel -c 2 python tools/profile_step.py --steps 2 > /tmp/ncu_$v.txt 2>&1
  echo "== $v" >> $out; grep -E "gpu__time|inst_executed|issue_active" /tmp/ncu_$v.txt | tail -3 >> $out
done
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:decode_kernel -c 2 python tools/profile_step.py --steps 2 > /tmp/ncu_main.txt 2>&1
echo "== main" >> $out; grep -E "gpu__time|inst_executed|issue_active" /tmp/ncu_main.txt | tail -3 >> $out
cat $out
