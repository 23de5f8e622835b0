# VIEWSHED launch-parameter A/B: warps per CTA and observer sort-tile size
mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for c in c2 c5; do
  for w in 0 8 16; do
    if [ $w = 0 ]; then unset TXS_VS_WARPS; else export TXS_VS_WARPS=$w; fi
    python profiles/scripts/stage_time.py $c viewshed 1 2>&1 | tail -1 | sed "s/^/warps=$w /" >> $O
  done
  unset TXS_VS_WARPS
  for t in 5 7 8; do
    TXS_VS_TILE_SHIFT=$t python profiles/scripts/stage_time.py $c viewshed 1 2>&1 | tail -1 | sed "s/^/tshift=$t /" >> $O
  done
done
