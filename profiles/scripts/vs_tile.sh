#!/bin/bash
# VIEWSHED observer sort tile (TXS_VS_TILE_SHIFT: 2^s-post square tiles)
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3 c5}; do
  for t in ${SHIFTS:-4 5 6}; do TXS_VS_TILE_SHIFT=$t python profiles/scripts/stage_time.py $c viewshed ${REPS:-2} | tail -1 | sed "s/^/$c tile_shift=$t /"; done
done
