#!/bin/bash
# VIX tile traversal (TXS_VIX_STRIP: strips of n 8x8-tile columns; default row-major at roi < 150, 16 at roi >= 150)
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3}; do
  python profiles/scripts/stage_time.py $c vix 3 | tail -1 | sed "s/^/default $c /"
  for s in ${STRIPS:-4 16 64 100000}; do
    TXS_VIX_STRIP=$s python profiles/scripts/stage_time.py $c vix 3 | tail -1 | sed "s/^/strip=$s $c /"
  done
done
