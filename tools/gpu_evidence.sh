#!/bin/bash
# round-2 evidence: K1 DRAM traffic (c2, c3), K1 ncu --set full (c2), launch lists (c2, c3 device-resident, shuffled, long journeys)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1800 python tools/decode_traffic.py c2 c3 > gpurun_out/traffic.log 2>&1
cp profiles/decode_traffic.json gpurun_out/decode_traffic.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -c 1 -o gpurun_out/k1_r02 python tools/profile_step.py --steps 1 --shards 128 > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_step.py --steps 1 --shards 128 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_step.py --steps 1 --journeys 1000000 --shards 128 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_shuf.csv python tools/profile_step.py --steps 1 --shuffle > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_long.csv python tools/profile_step.py --steps 1 --journeys 1000 --mean-duration 36000 > /dev/null 2>&1
cat gpurun_out/traffic.log
