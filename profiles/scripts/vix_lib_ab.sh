#!/bin/bash
# VIX stage ms per library variant (build/var/libtxsite_<name>.so; "default" = the release build)
cd "$(dirname "$0")/../.."
for v in ${VARS:-default}; do
  if [ $v != default ]; then export TXS_LIB=$PWD/build/var/libtxsite_$v.so; else unset TXS_LIB; fi
  for c in ${CFGS:-c3}; do echo "$v $c $(python profiles/scripts/stage_time.py $c vix 3 | tail -1)"; done
done
