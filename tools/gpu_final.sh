#!/bin/bash
# final evidence: smoke, reference arm (c3), default bench (c3), c2 bench, launch lists c2/c3
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
out=gpurun_out/final.log; : > $out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" >> $out 2>&1; echo "smoke rc=$?" >> $out
timeout 1200 python bench.py --impl reference --steps 8 --warmup 1 > gpurun_out/bench_ref_c3.log 2>&1; echo "ref rc=$?" >> $out
timeout 1500 python bench.py > gpurun_out/bench_c3_final.log 2>&1; echo "bench rc=$?" >> $out
timeout 900 python bench.py --workload c2 --steps 20 > gpurun_out/bench_c2_final.log 2>&1; echo "bench c2 rc=$?" >> $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_step.py --steps 1 --shards 128 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_step.py --steps 1 --journeys 1000000 --shards 128 > /dev/null 2>&1
cat $out; for f in bench_ref_c3 bench_c3_final bench_c2_final; do grep '^{' gpurun_out/$f.log | tail -1 | cut -c1-300; done
