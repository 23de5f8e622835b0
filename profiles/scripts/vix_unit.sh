#!/bin/bash
# VIX flattened skip test: groups per lane unit (VIX_UNIT) A/B, build/var/libtxsite_u*.so
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for v in ${VARS:-u2 u8}; do
  export TXS_LIB=$PWD/build/var/libtxsite_$v.so
  python -m pytest tests -m gpu -x -q -k "vix_skip" 2>&1 | tail -1 | sed "s/^/$v test: /" >> $O
  for c in c1 c2 c3; do python profiles/scripts/stage_time.py $c vix 3 2>&1 | tail -1 | sed "s/^/$v /" >> $O; done
done
unset TXS_LIB
for c in c1 c2 c3; do python profiles/scripts/stage_time.py $c vix 3 2>&1 | tail -1 | sed "s/^/default /" >> $O; done
