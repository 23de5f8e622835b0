#!/bin/bash
# SITE streaming gain pass: density-sized buckets (k_gain_tiled, default) vs TXS_GAIN_REG=1 (k_gain_full)
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3 c4 c5}; do
  python profiles/scripts/gain_once.py $c | tail -1 | sed "s/^/$c tiled-buckets /"
  TXS_GAIN_REG=1 python profiles/scripts/gain_once.py $c | tail -1 | sed "s/^/$c k_gain_full /"
done
