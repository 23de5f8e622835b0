#!/bin/bash
# VIX skip-test group size / unit A/B (TXS_VIX_GROUP, TXS_VIX_UNIT), min of 3 runs
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c1 c2 c3}; do
  for gu in "4 4" "4 8" "16 1" "16 2"; do
    set -- $gu
    TXS_VIX_GROUP=$1 TXS_VIX_UNIT=$2 python profiles/scripts/stage_time.py $c vix 3 | tail -1 | sed "s/^/$c G=$1 U=$2 /"
  done
done
