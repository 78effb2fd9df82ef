#!/bin/bash
# ring geometry sweep (c2) and the best candidates end to end at c3 (bench e2e only)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
out=gpurun_out/ingest2.log; : > $out
timeout 600 python tools/ring_sweep.py --reps 5 --grid "${GRID:-1:32,2:16,2:32,4:8,4:16,4:24,6:16}" --threads ${READERS:-8,10,12,16} >> $out 2>&1
for cfg in ${C3CFG:-4:16:12 2:16:12 32:16:16}; do
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
cat $out
