# VIEWSHED warps-per-CTA sweep (TXS_VS_WARPS)
mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for w in 15 18 20 24 32; do TXS_VS_WARPS=$w python profiles/scripts/stage_time.py c5 viewshed 1 2>&1 | tail -1 | sed "s/^/warps=$w /" >> $O; done
for w in 6 9 10; do TXS_VS_WARPS=$w python profiles/scripts/stage_time.py c2 viewshed 1 2>&1 | tail -1 | sed "s/^/warps=$w /" >> $O; done
for w in 6 8 12 16; do TXS_VS_WARPS=$w python profiles/scripts/stage_time.py c3 viewshed 1 2>&1 | tail -1 | sed "s/^/warps=$w /" >> $O; done
