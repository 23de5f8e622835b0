#!/bin/bash
# A/B of a stage between the default build and build/var/libtxsite_$VAR.so, alternating runs:
# VAR=vprev STAGE=vix CFGS="c2 c3" bash profiles/scripts/ab_stage.sh
cd "$(dirname "$0")/../.."
for rep in 1 2; do
  for c in ${CFGS:-c2 c3}; do
    python profiles/scripts/stage_time.py $c ${STAGE:-vix} 3 | tail -1 | sed "s/^/default $c /"
    TXS_LIB=$PWD/build/var/libtxsite_$VAR.so python profiles/scripts/stage_time.py $c ${STAGE:-vix} 3 | tail -1 | sed "s/^/$VAR $c /"
  done
done
