#!/bin/bash
# stage times for the default build and several build/var variants (VARS), alternating
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3}; do
  python profiles/scripts/stage_time.py $c ${STAGE:-vix} 3 | tail -1 | sed "s/^/default $c /"
  for v in $VARS; do
    TXS_LIB=$PWD/build/var/libtxsite_$v.so python profiles/scripts/stage_time.py $c ${STAGE:-vix} 3 | tail -1 | sed "s/^/$v $c /"
  done
done
