#!/bin/bash
# A/B of an environment switch: profile_step ARGS with and without ENV (e.g. CVLG_FOLD_GROUPS=1)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
out=gpurun_out/envab.log; : > $out
ENV=$1; shift
for a in "$@"; do
  echo "== base [$a]: $(timeout 900 python tools/profile_step.py $a 2>&1 | tail -1)" >> $out
  echo "== $ENV [$a]: $(env $ENV timeout 900 python tools/profile_step.py $a 2>&1 | tail -1)" >> $out
done
cat $out
