#!/bin/bash
# A/B of an environment knob on the VIX kernel time (bench.py, 3 steps).
#   usage (under gpurun): profiles/scripts/vix_env_ab.sh "c3 c2" VAR "v1 v2 ..."
O=gpurun_out; mkdir -p $O; rm -f $O/envab.txt
for c in $1; do for v in $3; do
  env $2=$v timeout 300 python bench.py --config $c --no-cpu-baseline --steps 3 > $O/envab_${c}_$v.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('$O/envab_${c}_$v.log') if l.startswith('{')][-1]); s=d['stages']['vix']
print('$c $2=$v', s['kernel_ms'], d['value'])" >> $O/envab.txt 2>&1
done; done
