#!/bin/bash
# VIEWSHED observers per CTA (TXS_VS_K) x warps per CTA (TXS_VS_WARPS) sweep
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c5}; do
  for kw in ${KW:-2:0 3:0 3:10 3:12 3:15}; do
    k=${kw%%:*}; w=${kw#*:}
    if [ $w = 0 ]; then TXS_VS_K=$k python profiles/scripts/stage_time.py $c viewshed 2 | tail -1 | sed "s/^/$c K=$k W=default /";
    else TXS_VS_K=$k TXS_VS_WARPS=$w python profiles/scripts/stage_time.py $c viewshed 2 | tail -1 | sed "s/^/$c K=$k W=$w /"; fi
  done
done
