mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for c in c1 c2 c3 c5; do
  python profiles/scripts/stage_time.py $c site 1 2>&1 | tail -1 | sed "s/^/default /" >> $O
  TXS_SITE_GRAPH=1 python profiles/scripts/stage_time.py $c site 1 2>&1 | tail -1 | sed "s/^/graph /" >> $O
done
