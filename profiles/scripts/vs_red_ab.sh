#!/bin/bash
# VIEWSHED cell-bit reds: predicated per observer (default) / one branch per cell event around K
# unconditional reds (VS_RED_GROUP=1) / the branch only when some observer sees the cell (2).
# Build first: profiles/scripts/build_variant.sh vsred1 viewshed -DVS_RED_GROUP=1 (and 2).
cd "$(dirname "$0")/../.."
for v in default vsred1 vsred2; do
  if [ $v != default ]; then export TXS_LIB=$PWD/build/var/libtxsite_$v.so; else unset TXS_LIB; fi
  for c in ${CFGS:-c3 c2 c5}; do
    echo "$v $c $(python profiles/scripts/stage_time.py $c viewshed 2 | tail -1)"
  done
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "viewshed" 2>&1 | tail -1
done
