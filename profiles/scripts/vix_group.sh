#!/bin/bash
# VIX skip-test group size / unit A/B (TXS_VIX_GROUP, TXS_VIX_UNIT), min of 3 runs
# GU="4:8 8:4" CFGS="c2 c3" bash profiles/scripts/vix_group.sh
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c1 c2 c3}; do
  for gu in ${GU:-4:4 4:8 16:1 16:2}; do
    g=${gu%%:*}; u=${gu#*:}
    TXS_VIX_GROUP=$g TXS_VIX_UNIT=$u python profiles/scripts/stage_time.py $c vix 3 | tail -1 | sed "s/^/$c G=$g U=$u /"
  done
done
