#!/bin/bash
# timings + launch lists of the secondary paths: shuffled c2 (full sort), long journeys, c5 shape
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
out=gpurun_out/paths.log; : > $out
echo "== c2" >> $out; timeout 300 python tools/profile_step.py --steps 6 >> $out 2>&1
echo "== c2 shuffled" >> $out; timeout 300 python tools/profile_step.py --steps 6 --shuffle >> $out 2>&1
echo "== long journeys (1000 x mean 36000 s)" >> $out; timeout 300 python tools/profile_step.py --steps 4 --journeys 1000 --mean-duration 36000 >> $out 2>&1
echo "== c5 shape (7 days fine)" >> $out; timeout 600 python tools/profile_step.py --steps 3 --days 7 --fine >> $out 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_shuf.csv python tools/profile_step.py --steps 1 --shuffle > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_long.csv python tools/profile_step.py --steps 1 --journeys 1000 --mean-duration 36000 > /dev/null 2>&1
cat $out
