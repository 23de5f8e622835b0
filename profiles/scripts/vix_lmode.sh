#!/bin/bash
# VIX k_vix_lanes variants (TXS_VIX_LMODE = mask | lazy << 1), stage ms per config.
#   usage (under gpurun): profiles/scripts/vix_lmode.sh c1 c2 c3 c4
O=gpurun_out; mkdir -p $O
for c in "$@"; do for m in 0 1 2 3; do
  TXS_VIX_LMODE=$m timeout 400 python bench.py --config $c --no-cpu-baseline --steps 3 > $O/lmode_${c}_$m.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('$O/lmode_${c}_$m.log') if l.startswith('{')][-1]); s=d['stages']['vix']
print('$c lmode $m vix kernel ms', s['kernel_ms'])" >> $O/lmode.txt
done; done
