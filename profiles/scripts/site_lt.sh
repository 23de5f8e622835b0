#!/bin/bash
# persistent SITE loop: threads per CTA (SITE_LOOP_THREADS builds) x CTAs per SM (TXS_SITE_LOOP_CTAS)
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3}; do
  python profiles/scripts/stage_time.py $c site 3 | tail -1 | sed "s/^/default $c /"
  for v in lt512:1 lt512:2 lt1024:1; do
    b=${v%%:*}; k=${v#*:}
    TXS_SITE_LOOP_CTAS=$k TXS_LIB=$PWD/build/var/libtxsite_$b.so python profiles/scripts/stage_time.py $c site 3 | tail -1 | sed "s/^/$b x$k $c /"
  done
done
