#!/bin/bash
# per-candidate gain pass: CTAs per SM of the grid (TXS_GAIN_GRID) x layout
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3 c4 c5}; do
  for g in ${GRIDS:-5 10 16 64 256}; do
    TXS_GAIN_GRID=$g timeout 900 python profiles/scripts/gain_kinds.py $c full t8 2>&1 | tail -2 | sed "s/^/grid=$g /"
  done
done
