#!/bin/bash
# persistent VIX grid sweep (TXS_VIX_GRID; default = resident CTAs = 4 x SMs)
cd "$(dirname "$0")/../.."
for g in 0 1184 296; do
  echo "grid $g"
  for c in c2 c3; do
    if [ $g = 0 ]; then python profiles/scripts/stage_time.py $c vix 3 | tail -1; else TXS_VIX_GRID=$g python profiles/scripts/stage_time.py $c vix 3 | tail -1; fi
  done
done
