#!/bin/bash
# A/B of build_variant.sh libraries on the VIX kernel time (bench.py, 3 steps).
#   usage (under gpurun): profiles/scripts/vix_ab_libs.sh "c3 c2" "default minb3 ..."
O=gpurun_out; mkdir -p $O; rm -f $O/ab.txt
for c in $1; do for lib in $2; do
  if [ $lib = default ]; then unset TXS_LIB; else export TXS_LIB=build/var/libtxsite_$lib.so; fi
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 3 > $O/ab_${c}_$lib.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('$O/ab_${c}_$lib.log') if l.startswith('{')][-1]); s=d['stages']['vix']
print('$c $lib', s['kernel_ms'], d['value'])" >> $O/ab.txt 2>&1
done; done
