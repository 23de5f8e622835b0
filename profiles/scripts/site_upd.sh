mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for m in 16 24 32 64; do TXS_UPD_MULT=$m python profiles/scripts/stage_time.py c5 site 1 2>&1 | tail -1 | sed "s/^/upd=$m /" >> $O; done
for m in 8 16 32; do TXS_UPD_MULT=$m TXS_SITE_GRAPH=1 python profiles/scripts/stage_time.py c3 site 1 2>&1 | tail -1 | sed "s/^/graph upd=$m /" >> $O; done
