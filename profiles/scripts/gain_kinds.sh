#!/bin/bash
# SITE streaming gain pass A/B: per-candidate / bucket-tiled / strip-tile forms, strip-tile shapes
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3 c4 c5}; do
  timeout 600 python profiles/scripts/gain_kinds.py $c full tiled strips 2>&1 | tail -3
  for shtx in ${SHAPES:-16x8 32x4 32x16 64x8}; do
    sh=${shtx%x*}; tx=${shtx#*x}
    TXS_STRIP_ROWS=$sh TXS_STRIP_TX=$tx timeout 600 python profiles/scripts/gain_kinds.py $c strips 2>&1 | tail -1 | sed "s/^/SH=$sh TX=$tx /"
  done
done
