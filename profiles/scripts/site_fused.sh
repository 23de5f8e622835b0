mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
TXS_SITE_FUSED=1 python -m pytest tests -m gpu -x -q -k "site or shard" 2>&1 | tail -1 | sed "s/^/fused test: /" >> $O
for c in c1 c2 c3; do for v in 0 1; do TXS_SITE_FUSED=$v python profiles/scripts/stage_time.py $c site 2 2>&1 | tail -1 | sed "s/^/fused=$v /" >> $O; done; done
for v in 0 1; do TXS_SITE_FUSED=$v python profiles/scripts/stage_time.py c4 site 1 2>&1 | tail -1 | sed "s/^/fused=$v /" >> $O; done
