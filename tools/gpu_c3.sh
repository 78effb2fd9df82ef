#!/bin/bash
# c3 evidence: full-trace parity against the reference, ring geometry at c3, the default bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
out=gpurun_out/c3.log; : > $out
timeout 1500 python tools/c3_parity.py >> $out 2>&1
for cfg in ${C3CFG:-4:16:10 6:16:10 8:16:10 4:24:10 4:16:8 4:16:12}; do
  IFS=: read mb sl rd <<< "$cfg"
  echo "== c3 e2e ring $mb MB x $sl slots, $rd readers" >> $out
  CVLG_RING_MB=$mb CVLG_RING_SLOTS=$sl CVLG_RING_READERS=$rd timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-parity > /tmp/b.log 2>&1
  python -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print(d['e2e']['ms_per_step'], d['e2e']['value']/1e9, 'G rec/s e2e; device ms', d['ms_per_step']) if d else print(open('/tmp/b.log').read()[-1500:])
" >> $out
done
timeout 1200 python bench.py > gpurun_out/bench_c3_default.log 2>&1
tail -c 3000 gpurun_out/bench_c3_default.log >> $out
cat $out
