#!/bin/bash
# SITE streaming gain pass: cum-aligned rows / bucket-tiled / 8x8-tile shadow layout
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3 c4 c5}; do
  timeout 900 python profiles/scripts/gain_kinds.py $c full tiled t8 2>&1 | tail -3
done
